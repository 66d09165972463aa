# iteration pass: parity subset, host-API tests, config-2 levels, ncu of the L13 solves, drop-in e2e
TAG=${1:-r2e}
O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity_full.py -k "targeted or config2" -x -q -p no:cacheprovider > $O/parity.log 2>&1; echo rc=$? >> $O/parity.log
timeout 900 python -m pytest tests/test_capi.py tests/test_gpu_parity.py tests/test_dropin_gpu.py tests/test_cpp_shim.py tests/test_container.py tests/test_compress.py -m gpu -x -q -p no:cacheprovider > $O/hosttests.log 2>&1; echo rc=$? >> $O/hosttests.log
timeout 300 python profiles/scripts/levels.py --shape 8193,8193 --dtype float64 > $O/levels_cfg2.txt 2>&1
g++ -std=c++17 -O2 -Iinclude tests/cpp/bench_dropin.cpp -Lpaper_2105_12764_b200 -lmgrg -pthread -Wl,-rpath,$PWD/paper_2105_12764_b200 -o /tmp/bench_dropin
timeout 300 /tmp/bench_dropin 1025 3 1 0 > $O/dropin.jsonl 2>&1
timeout 300 /tmp/bench_dropin 1025 3 1 1 >> $O/dropin.jsonl 2>&1
bash profiles/scripts/ncu_one.sh thomas_cluster 0 ${TAG}_c2x --shape 8193,8193 --dtype float64
bash profiles/scripts/ncu_one.sh thomas_cluster 1 ${TAG}_c2y --shape 8193,8193 --dtype float64
