TAG=${1:-r2ao}
O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_units.py tests/test_container.py tests/test_compress.py tests/test_cpp_shim.py -x -q -p no:cacheprovider > $O/parity.log 2>&1; echo rc=$? >> $O/parity.log
timeout 300 python profiles/scripts/levels.py --shape 129,129,129,9 > $O/levels_4d.txt 2>&1
timeout 300 python profiles/scripts/bench_widen.py > $O/widen.json 2>&1
