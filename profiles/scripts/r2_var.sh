TAG=${1:-r2t}
O=gpurun_out/$TAG; mkdir -p $O
for v in base nw8f32; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2105_12764_b200/variants/libmgrg_$v.so; fi
  MGRG_LIB=$L timeout 300 python profiles/scripts/levels.py > $O/levels_c4_$v.txt 2>&1
done
MGRG_LIB=$PWD/paper_2105_12764_b200/variants/libmgrg_nw8f32.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "fast" > $O/parity_nw8.log 2>&1; echo rc=$? >> $O/parity_nw8.log
