O=gpurun_out/${1:-r2crc}
mkdir -p $O
timeout 300 python profiles/scripts/crc_time.py > $O/crc_v2.json 2>&1
MGRG_LIB=paper_2105_12764_b200/variants/libmgrg_knobs.so MGRG_CRC_V2=0 timeout 300 python profiles/scripts/crc_time.py > $O/crc_v1.json 2>&1
timeout 600 python -m pytest tests/test_container.py tests/test_compress.py -x -q -p no:cacheprovider > $O/tests.log 2>&1; echo rc=$? >> $O/tests.log
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none --csv -k regex:crc_ --log-file $O/crc_list.csv python profiles/scripts/crc_time.py > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none -k regex:crc_blocks2 -s 2 -c 1 -o $O/crc2 python profiles/scripts/crc_time.py > /dev/null 2>&1
