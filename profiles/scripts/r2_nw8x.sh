O=gpurun_out/r2nw8x
mkdir -p $O
V=paper_2105_12764_b200/variants/libmgrg_nw8x.so
MGRG_LIB=$V timeout 900 python -m pytest tests/test_gpu_parity_full.py -x -q -p no:cacheprovider -k "targeted or config2" > $O/parity.log 2>&1; echo rc=$? >> $O/parity.log
MGRG_LIB=$V timeout 300 python profiles/scripts/levels.py --shape 8193,8193 --dtype float64 > $O/levels_c2_nw8x.txt 2>&1
timeout 300 python profiles/scripts/levels.py --shape 8193,8193 --dtype float64 > $O/levels_c2_base.txt 2>&1
