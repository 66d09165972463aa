# Two-pass long-fiber Thomas: parity of the long-fiber shapes + config-2 A/B (levels) + launch list.
O=gpurun_out/${1:-r2tp}
mkdir -p $O
V=paper_2105_12764_b200/variants/libmgrg_knobs.so
timeout 900 python -m pytest tests/test_gpu_parity_full.py -x -q -p no:cacheprovider -k "targeted or config2" > $O/parity.log 2>&1; echo rc=$? >> $O/parity.log
for t in 100000 4097; do
  MGRG_LIB=$V MGRG_TP_MIN=$t timeout 300 python profiles/scripts/levels.py --shape 8193,8193 --dtype float64 > $O/levels_c2_tp$t.txt 2>&1
done
timeout 300 python profiles/scripts/levels.py --shape 8193,8193 --dtype float64 > $O/levels_c2_release.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none --csv -k regex:"tp_|thomas" --log-file $O/tp_list.csv python profiles/scripts/tp_probe.py > /dev/null 2>&1
ls -la $O
