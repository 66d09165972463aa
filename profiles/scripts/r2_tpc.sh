O=gpurun_out/r2tpc
mkdir -p $O
for v in c8 c32; do
  MGRG_LIB=paper_2105_12764_b200/variants/libmgrg_$v.so timeout 600 python -m pytest tests/test_gpu_parity_full.py -x -q -p no:cacheprovider -k "targeted" > $O/parity_$v.log 2>&1; echo rc=$? >> $O/parity_$v.log
  MGRG_LIB=paper_2105_12764_b200/variants/libmgrg_$v.so timeout 300 python profiles/scripts/levels.py --shape 8193,8193 --dtype float64 > $O/levels_c2_$v.txt 2>&1
done
timeout 300 python profiles/scripts/levels.py --shape 8193,8193 --dtype float64 > $O/levels_c2_base.txt 2>&1
