TAG=${1:-r2u}
O=gpurun_out/$TAG; mkdir -p $O
for v in base cl16; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2105_12764_b200/variants/libmgrg_$v.so; fi
  MGRG_LIB=$L timeout 300 python profiles/scripts/levels.py --shape 8193,8193 --dtype float64 > $O/levels_c2_$v.txt 2>&1
done
MGRG_LIB=$PWD/paper_2105_12764_b200/variants/libmgrg_cl16.so timeout 600 python -m pytest tests/test_gpu_parity_full.py -x -q -p no:cacheprovider -k "targeted or config2" > $O/parity_cl16.log 2>&1; echo rc=$? >> $O/parity_cl16.log
