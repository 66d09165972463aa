TAG=${1:-r2be}
O=gpurun_out/$TAG; mkdir -p $O
for v in base t3m4 t2m4 t2m5; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2105_12764_b200/variants/libmgrg_$v.so; fi
  MGRG_LIB=$L timeout 300 python profiles/scripts/levels.py > $O/levels_c4_$v.txt 2>&1
done
