O=gpurun_out/r2persist
mkdir -p $O
V=paper_2105_12764_b200/variants/libmgrg_persist.so
MGRG_LIB=$V timeout 600 python -m pytest tests/test_gpu_parity_full.py -x -q -p no:cacheprovider -k "targeted" > $O/parity.log 2>&1; echo rc=$? >> $O/parity.log
MGRG_LIB=$V timeout 300 python profiles/scripts/levels.py > $O/levels_persist.txt 2>&1
timeout 300 python profiles/scripts/levels.py > $O/levels_base.txt 2>&1
