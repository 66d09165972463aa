O=gpurun_out/r2zw
mkdir -p $O
for r in 1 2; do
for v in zw16 zw64; do
  MGRG_LIB=paper_2105_12764_b200/variants/libmgrg_$v.so timeout 300 python profiles/scripts/levels.py > $O/levels_${v}_$r.txt 2>&1
done
timeout 300 python profiles/scripts/levels.py > $O/levels_base_$r.txt 2>&1
done
