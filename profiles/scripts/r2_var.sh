TAG=${1:-r2bb}
O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py -k "not config4 and not config5_block and not config3" -x -q -p no:cacheprovider > $O/t.log 2>&1; echo rc=$? >> $O/t.log
for v in base head; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2105_12764_b200/variants/libmgrg_$v.so; fi
  MGRG_LIB=$L timeout 300 python profiles/scripts/levels.py > $O/levels_c4_$v.txt 2>&1
  MGRG_LIB=$L timeout 300 python profiles/scripts/levels.py --shape 1025,1025,513 --dtype float64 > $O/levels_c5_$v.txt 2>&1
done
