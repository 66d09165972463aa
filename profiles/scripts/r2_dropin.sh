TAG=${1:-r2g}
O=gpurun_out/$TAG; mkdir -p $O
g++ -std=c++17 -O2 -Iinclude tests/cpp/bench_dropin.cpp -Lpaper_2105_12764_b200 -lmgrg -pthread -Wl,-rpath,$PWD/paper_2105_12764_b200 -o /tmp/bench_dropin
timeout 300 /tmp/bench_dropin 1025 2 1 1 > $O/dropin.jsonl 2>&1
nproc >> $O/dropin.jsonl; free -g >> $O/dropin.jsonl; cat /sys/kernel/mm/transparent_hugepage/enabled >> $O/dropin.jsonl; uname -r >> $O/dropin.jsonl
