TAG=${1:-r2af}
O=gpurun_out/$TAG; mkdir -p $O
timeout 300 python profiles/scripts/tail_probe.py > $O/tail.json 2>&1
