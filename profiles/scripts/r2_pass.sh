# Round-2 GPU pass: gpu tests, bench line (+ graphs A/B), reference arm, launch list.
TAG=${1:-r2a}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo rc=$? >> $O/gputest.log
timeout 600 python bench.py > $O/bench.jsonl 2>$O/bench.err
timeout 600 python bench.py --graphs --no-cpu --no-others >> $O/bench.jsonl 2>>$O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 >> $O/bench.jsonl 2>>$O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-others > /dev/null 2>&1
timeout 600 python profiles/scripts/levels.py > $O/levels.txt 2>&1
ls -la $O
