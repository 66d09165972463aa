TAG=${1:-r2l}
O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py -x -q -p no:cacheprovider > $O/parity.log 2>&1; echo rc=$? >> $O/parity.log
for v in base rlf32m2 rlf32t8m2; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2105_12764_b200/variants/libmgrg_$v.so; fi
  MGRG_LIB=$L timeout 300 python profiles/scripts/levels.py > $O/levels_c4_$v.txt 2>&1
done
bash profiles/scripts/ncu_one.sh lean_dec 0 ${TAG}_ldec
