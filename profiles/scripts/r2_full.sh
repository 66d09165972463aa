# full pass: all GPU tests, bench line (with drop-in e2e), config-2 levels, launch list
TAG=${1:-r2f}
O=gpurun_out/$TAG; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo rc=$? >> $O/gputest.log
timeout 900 python bench.py > $O/bench.jsonl 2>$O/bench.err
timeout 300 python profiles/scripts/levels.py --shape 8193,8193 --dtype float64 > $O/levels_cfg2.txt 2>&1
timeout 300 python profiles/scripts/levels.py > $O/levels.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-others > /dev/null 2>&1
