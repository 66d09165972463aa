TAG=${1:-r2z}
O=gpurun_out/$TAG; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_coop.py -x -q -p no:cacheprovider > $O/parity.log 2>&1; echo rc=$? >> $O/parity.log
timeout 300 python profiles/scripts/levels.py > $O/levels_c4.txt 2>&1
timeout 300 python profiles/scripts/levels.py --shape 1025,1025,513 --dtype float64 > $O/levels_c5.txt 2>&1
timeout 300 python profiles/scripts/levels.py --exact > $O/levels_c4x.txt 2>&1
bash profiles/scripts/ncu_one.sh lean_dec 0 ${TAG}_ldec
