# late round-2 pass: sanitizer on the new kernels, full GPU suite, smoke, bench, launch list, levels
O=gpurun_out/${1:-r2fin}
mkdir -p $O
# (compute-sanitizer is closed on this pool: see profiles/r2/late/sanitizer_closed.txt)
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo rc=$? >> $O/gputest.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo rc=$? >> $O/smoke.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 600 python bench.py > $O/bench.jsonl 2>$O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 >> $O/bench.jsonl 2>>$O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-others > /dev/null 2>&1
timeout 600 python profiles/scripts/levels.py > $O/levels.txt 2>&1
timeout 600 python profiles/scripts/levels.py --shape 8193,8193 --dtype float64 > $O/levels_cfg2.txt 2>&1
timeout 300 python profiles/scripts/crc_time.py > $O/crc.json 2>&1
ls -la $O
