TAG=${1:-r2bh}
O=gpurun_out/$TAG; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo rc=$? >> $O/gputest.log
timeout 300 python profiles/scripts/levels.py --exact > $O/levels_c4x.txt 2>&1
timeout 300 python profiles/scripts/levels.py --exact --shape 1025,1025,513 --dtype float64 > $O/levels_c5x.txt 2>&1
timeout 300 python profiles/scripts/levels.py > $O/levels_c4.txt 2>&1
