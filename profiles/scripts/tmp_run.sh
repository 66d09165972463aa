python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/t8.log 2>&1; echo rc=$? >> gpurun_out/t8.log
python bench.py --steps 50 --warmup 5 --no-cpu --no-others > gpurun_out/bench8.jsonl 2> gpurun_out/bench8.err
python profiles/scripts/levels.py > gpurun_out/lv_base.txt 2>&1
