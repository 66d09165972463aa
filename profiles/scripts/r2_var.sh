TAG=${1:-r2bk}
O=gpurun_out/$TAG; mkdir -p $O
for v in base b16 b32; do
  if [ $v = base ]; then L=""; else L=$PWD/paper_2105_12764_b200/variants/libmgrg_$v.so; fi
  MGRG_LIB=$L timeout 300 python profiles/scripts/levels.py --exact > $O/levels_c4x_$v.txt 2>&1
done
