TAG=${1:-r2ba}
O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests/test_dropin_gpu.py tests/test_capi.py tests/test_cpp_shim.py -x -q -p no:cacheprovider > $O/t.log 2>&1; echo rc=$? >> $O/t.log
g++ -std=c++17 -O2 -Iinclude tests/cpp/bench_dropin.cpp -Lpaper_2105_12764_b200 -lmgrg -pthread -Wl,-rpath,$PWD/paper_2105_12764_b200 -o /tmp/bench_dropin
timeout 300 /tmp/bench_dropin 1025 2 1 0 > $O/dropin.jsonl 2>&1
timeout 300 /tmp/bench_dropin 1025 2 1 1 >> $O/dropin.jsonl 2>&1
