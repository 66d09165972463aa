O=gpurun_out/r2c2
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity_full.py -x -q -p no:cacheprovider -k "targeted or config2" > $O/parity.log 2>&1; echo rc=$? >> $O/parity.log
timeout 300 python profiles/scripts/levels.py --shape 8193,8193 --dtype float64 > $O/levels_c2.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv -k regex:"tp_" --log-file $O/list.csv python profiles/scripts/tp_probe.py > /dev/null 2>&1
