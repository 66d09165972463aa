TAG=${1:-r2o}
O=gpurun_out/$TAG; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo rc=$? >> $O/gputest.log
timeout 300 python profiles/scripts/levels.py --shape 1025,1025,513 --dtype float64 > $O/levels_c5.txt 2>&1
timeout 300 python profiles/scripts/levels.py --shape 8193,8193 --dtype float64 > $O/levels_c2.txt 2>&1
timeout 300 python profiles/scripts/levels.py --shape 513,513,513 > $O/levels_c3u.txt 2>&1
