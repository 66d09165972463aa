O=gpurun_out/${1:-r2tpn}
mkdir -p $O
V=paper_2105_12764_b200/variants/libmgrg_knobs.so
MGRG_LIB=$V MGRG_TP_MIN=1025 timeout 120 python profiles/scripts/tp_probe.py > $O/probe.log 2>&1
MGRG_LIB=$V MGRG_TP_MIN=1025 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none --csv -k regex:"tp_|thomas" --log-file $O/tp_list.csv python profiles/scripts/tp_probe.py > /dev/null 2>&1
MGRG_LIB=$V MGRG_TP_MIN=1025 timeout 600 ncu --set full --import-source on --clock-control none -k regex:tp_pass -c 4 -o $O/tp_full python profiles/scripts/tp_probe.py > $O/ncu_full.log 2>&1
ls -la $O
