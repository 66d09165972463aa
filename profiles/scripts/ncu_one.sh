# Full ncu capture of ONE kernel launch of profile_step.py (1025^3 f32 FAST),
# exported to CSV (raw + details + SASS source) under gpurun_out/.
#   bash profiles/scripts/ncu_one.sh <name-regex> <launch-skip> <tag> [profile_step args]
K=$1; SKIP=$2; TAG=$3; shift 3
rm -f gpurun_out/$TAG.ncu-rep
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K --launch-skip $SKIP -c 1 \
  -o gpurun_out/$TAG python profiles/profile_step.py --fast "$@" > gpurun_out/$TAG.log 2>&1
ncu -i gpurun_out/$TAG.ncu-rep --page raw --csv > gpurun_out/$TAG.raw.csv 2>/dev/null
ncu -i gpurun_out/$TAG.ncu-rep --page details --csv > gpurun_out/$TAG.details.csv 2>/dev/null
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source sass > gpurun_out/$TAG.sass.csv 2>/dev/null
ncu -i gpurun_out/$TAG.ncu-rep --page source --csv --print-source cuda > gpurun_out/$TAG.cuda.csv 2>/dev/null
gzip -f gpurun_out/$TAG.sass.csv gpurun_out/$TAG.cuda.csv
mkdir -p /tmp/reps && mv gpurun_out/$TAG.ncu-rep /tmp/reps/
