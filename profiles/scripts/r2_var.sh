TAG=${1:-r2ac}
O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_full.py tests/test_cpp_shim.py -x -q -p no:cacheprovider > $O/parity.log 2>&1; echo rc=$? >> $O/parity.log
timeout 300 python profiles/scripts/levels.py --exact > $O/levels_c4x.txt 2>&1
