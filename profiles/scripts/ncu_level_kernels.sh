# Full ncu captures of the 1025^3 f32 level kernels (one launch each, L10).
# Run on the GPU box: bash profiles/scripts/ncu_level_kernels.sh
set -x
rm -f gpurun_out/*.ncu-rep
P="python profiles/profile_step.py --fast"
NCU="ncu --set full --clock-control none --import-source on"
timeout 600 $NCU -k regex:dec4_kernel -c 1 -o gpurun_out/r1s3_dec4 $P > gpurun_out/ncu_dec4.log 2>&1
timeout 600 $NCU -k regex:rl2_kernel --launch-skip 9 -c 1 -o gpurun_out/r1s3_rl2 $P > gpurun_out/ncu_rl2.log 2>&1
timeout 600 $NCU -k regex:rg2_kernel --launch-skip 9 -c 1 -o gpurun_out/r1s3_rg2 $P > gpurun_out/ncu_rg2.log 2>&1
timeout 600 $NCU -k regex:thomas -c 3 -o gpurun_out/r1s3_thomas $P > gpurun_out/ncu_thomas.log 2>&1
ls -la gpurun_out
# summaries (the .ncu-rep files exceed gpurun's 64 MiB return limit)
for r in gpurun_out/r1s3_*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > $b.sass.csv 2>/dev/null
  gzip -f $b.sass.csv
done
mkdir -p /tmp/reps && mv gpurun_out/*.ncu-rep /tmp/reps/
du -sh gpurun_out
