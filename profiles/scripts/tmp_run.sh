python -m pytest tests/test_dropin_gpu.py -x -q -p no:cacheprovider > gpurun_out/t9.log 2>&1; echo rc=$? >> gpurun_out/t9.log
for i in 1 2; do
python bench.py --steps 50 --warmup 5 --no-cpu --no-others --no-e2e > gpurun_out/b9_pdl_$i.jsonl 2>&1
python bench.py --steps 50 --warmup 5 --no-cpu --no-others --no-e2e --graphs > gpurun_out/b9_graph_$i.jsonl 2>&1
done
