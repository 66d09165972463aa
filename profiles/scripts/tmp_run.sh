python -m pytest tests/test_gpu_parity.py tests/test_coop.py -x -q -p no:cacheprovider > gpurun_out/t10.log 2>&1; echo rc=$? >> gpurun_out/t10.log
python profiles/scripts/levels.py > gpurun_out/lv_base.txt 2>&1
