O=gpurun_out/r2crc5
mkdir -p $O
timeout 600 python -m pytest tests/test_container.py tests/test_compress.py tests/test_dropin_gpu.py -x -q -p no:cacheprovider > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
for i in 1 2; do timeout 200 python profiles/scripts/crc_time.py >> $O/crc.json 2>&1; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:crc_ --log-file $O/crc_list.csv python profiles/scripts/crc_time.py > /dev/null 2>&1
