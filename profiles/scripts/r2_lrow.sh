# warp-per-fiber long x-fiber Thomas: parity + A/B (levels) for 8193^2 f64 / 4097^2 f32
O=gpurun_out/${1:-r2lr}
mkdir -p $O
V=paper_2105_12764_b200/variants/libmgrg_knobs.so
timeout 900 python -m pytest tests/test_gpu_parity_full.py -x -q -p no:cacheprovider -k "targeted or config2" > $O/parity.log 2>&1; echo rc=$? >> $O/parity.log
for t in 100000 1025 2049; do
  MGRG_LIB=$V MGRG_LROW_MIN=$t timeout 300 python profiles/scripts/levels.py --shape 8193,8193 --dtype float64 > $O/levels_c2_lr$t.txt 2>&1
  MGRG_LIB=$V MGRG_LROW_MIN=$t timeout 300 python profiles/scripts/levels.py --shape 4097,4097 --dtype float32 > $O/levels_4097f32_lr$t.txt 2>&1
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none --csv -k regex:"lrow|tp_|thomas" --log-file $O/list.csv python profiles/scripts/tp_probe.py > /dev/null 2>&1
ls $O
