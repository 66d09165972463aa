TAG=${1:-r2az}
O=gpurun_out/$TAG; mkdir -p $O
timeout 300 python profiles/scripts/tail_probe.py > $O/tail_base.json 2>&1
for v in ts24 ts8 ts0; do
MGRG_LIB=$PWD/paper_2105_12764_b200/variants/libmgrg_$v.so timeout 300 python profiles/scripts/tail_probe.py > $O/tail_$v.json 2>&1
done
