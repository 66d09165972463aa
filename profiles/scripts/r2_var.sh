TAG=${1:-r2bi}
O=gpurun_out/$TAG; mkdir -p $O
for v in base e2m4 e2m5 e4m3 e4m4; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2105_12764_b200/variants/libmgrg_$v.so; fi
  MGRG_LIB=$L timeout 300 python profiles/scripts/levels.py --exact > $O/levels_c4x_$v.txt 2>&1
done
