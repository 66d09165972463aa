# Round-2 ncu pass: host-transfer probe, launch list of config 2, full captures of
# the L10 headline kernels and of config 2's long-fiber Thomas solves.
TAG=${1:-r2b}
mkdir -p gpurun_out/$TAG
./profiles/scripts/host_probe/host_probe > gpurun_out/$TAG/host_probe.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/$TAG/launches_cfg2.csv python profiles/profile_step.py --fast --shape 8193,8193 --dtype float64 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/$TAG/step_dram.csv python profiles/profile_step.py --fast > /dev/null 2>&1
for spec in "lean_dec 0 ldec" "lean_rload 9 lrl" "lean_rgpk 9 lrg" "thomas_fiber 1 tfy"; do
  set -- $spec
  bash profiles/scripts/ncu_one.sh $1 $2 ${TAG}_$3
done
bash profiles/scripts/ncu_one.sh thomas_fiber 0 ${TAG}_c2x --shape 8193,8193 --dtype float64
bash profiles/scripts/ncu_one.sh thomas_fiber 1 ${TAG}_c2y --shape 8193,8193 --dtype float64
