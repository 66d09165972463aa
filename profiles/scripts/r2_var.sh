TAG=${1:-r2aw}
O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests/test_dropin_gpu.py tests/test_capi.py tests/test_gpu_parity.py tests/test_cpp_shim.py -x -q -p no:cacheprovider > $O/t.log 2>&1; echo rc=$? >> $O/t.log
