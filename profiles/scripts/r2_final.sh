# Round-2 profile pass (1025^3 f32 FAST unless noted): bench line + reference arm, launch list,
# per-kernel DRAM of one dec+rec, full captures of the L10 kernels, level tables of every config.
TAG=${1:-r2final}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 900 python bench.py > $O/bench.jsonl 2>$O/bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 >> $O/bench.jsonl 2>>$O/bench.err
timeout 900 python bench.py --config 5 --steps 10 --warmup 3 >> $O/bench.jsonl 2>>$O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e --no-others > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $O/step_dram.csv python profiles/profile_step.py --fast > /dev/null 2>&1
for spec in "lean_dec 0 ldec" "lean_rload 9 lrl" "lean_rgpk 9 lrg" "thomas_fiber 0 tfx" "thomas_fiber 1 tfy" "thomas_fiber 2 tfz"; do
  set -- $spec
  bash profiles/scripts/ncu_one.sh $1 $2 ${TAG}_$3
done
for sh in "1025,1025,1025 float32" "513,513,513 float32" "8193,8193 float64" "1025,1025,513 float64" "65,65,65 float64"; do
  set -- $sh
  timeout 300 python profiles/scripts/levels.py --shape $1 --dtype $2 > $O/levels_$(echo $1 | tr , x)_$2.txt 2>&1
done
ls -la $O
