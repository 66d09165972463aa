TAG=${1:-r2h}
O=gpurun_out/$TAG; mkdir -p $O
timeout 600 python -m pytest tests/test_dropin_gpu.py -x -q -p no:cacheprovider > $O/dropin_tests.log 2>&1; echo rc=$? >> $O/dropin_tests.log
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 > $O/bench_c5.jsonl 2>$O/bench_c5.err
timeout 900 python bench.py --config 5 --impl reference --steps 1 --warmup 0 >> $O/bench_c5.jsonl 2>>$O/bench_c5.err
