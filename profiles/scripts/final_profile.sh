# Round artifacts on the GPU box (1025^3 f32, FAST): bench line, reference
# arm, launch list, per-kernel DRAM totals of one decompose + recompose, and
# full captures of the dominant L10 kernels.   bash profiles/scripts/final_profile.sh TAG
TAG=${1:-final}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt
timeout 600 python bench.py > $O/bench.jsonl 2>$O/bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 >> $O/bench.jsonl 2>>$O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $O/launches_bench.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file $O/step_dram.csv python profiles/profile_step.py --fast > /dev/null 2>&1
for spec in "lean_dec 0 ldec" "lean_rload 9 lrl" "lean_rgpk 9 lrg" "thomas_fiber 0 tfx" "thomas_fiber 1 tfy" "thomas_fiber 2 tfz"; do
  set -- $spec
  bash profiles/scripts/ncu_one.sh $1 $2 ${TAG}_$3
done
timeout 600 python profiles/scripts/levels.py > $O/levels.txt 2>&1
timeout 600 python profiles/scripts/bench_container.py > $O/container.json 2>/dev/null
timeout 600 python profiles/scripts/bench_compress.py > $O/compress.json 2>/dev/null
ls -la $O
