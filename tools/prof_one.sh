#!/bin/bash
# usage: tools/prof_one.sh <workload> [kernel-regex]  -- plain run, then one
# ncu --set full capture exported to CSV (raw / source) under gpurun_out/.
set -u
W=$1; K=${2:-"nchw|pool_|conv2d_|tc_"}
OUT=gpurun_out
timeout 120 python tools/prof_workload.py $W 1 > $OUT/plain_$W.log 2>&1 || { echo "plain run failed"; exit 1; }
timeout 900 ncu -f --set full --clock-control none --import-source on -k regex:"$K" -c ${NCU_COUNT:-1} \
    -o /tmp/prof_$W python tools/prof_workload.py $W 1 > $OUT/ncu_$W.log 2>&1
ncu -i /tmp/prof_$W.ncu-rep --page raw --csv > $OUT/raw_$W.csv 2>/dev/null
ncu -i /tmp/prof_$W.ncu-rep --page details --csv > $OUT/details_$W.csv 2>/dev/null
ncu -i /tmp/prof_$W.ncu-rep --page source --csv --print-source sass > $OUT/source_$W.csv 2>/dev/null
gzip -f $OUT/source_$W.csv
python tools/ncu_summary.py $OUT/raw_$W.csv
