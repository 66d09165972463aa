O=gpurun_out/${1:-r2tpx}
mkdir -p $O
V=paper_2105_12764_b200/variants/libmgrg_knobs.so
MGRG_LIB=$V MGRG_TP_X=1 timeout 900 python -m pytest tests/test_gpu_parity_full.py -x -q -p no:cacheprovider -k "targeted or config2" > $O/parity.log 2>&1; echo rc=$? >> $O/parity.log
for x in 0 1; do
  MGRG_LIB=$V MGRG_TP_X=$x timeout 300 python profiles/scripts/levels.py --shape 8193,8193 --dtype float64 > $O/levels_c2_x$x.txt 2>&1
done
MGRG_LIB=$V MGRG_TP_X=1 MGRG_TP_MIN=2049 timeout 300 python profiles/scripts/levels.py --shape 8193,8193 --dtype float64 > $O/levels_c2_x1_min2049.txt 2>&1
MGRG_LIB=$V MGRG_TP_X=1 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none --csv -k regex:"tp_|thomas" --log-file $O/list.csv python profiles/scripts/tp_probe.py > /dev/null 2>&1
