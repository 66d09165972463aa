TAG=${1:-r2aj}
O=gpurun_out/$TAG; mkdir -p $O
timeout 300 python profiles/scripts/bisect_exact.py paper_2105_12764_b200/libmgrg.so > $O/bisect.log 2>&1
timeout 600 python profiles/scripts/dbg_exact2d.py > $O/dbg.log 2>&1
timeout 900 python profiles/scripts/sanitize_cases.py > $O/cases_plain.log 2>&1; echo rc=$? >> $O/cases_plain.log
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $O/gputest.log 2>&1; echo rc=$? >> $O/gputest.log
