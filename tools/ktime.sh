#!/bin/bash
# usage: tools/ktime.sh <workload> <kernel-regex>: per-launch device time of one kernel
# family (ncu launch list, clock-control none), after a plain run exits 0.
W=$1; K=$2
timeout 120 python tools/prof_workload.py $W 3 > /dev/null 2>&1 || { echo "plain run failed"; exit 1; }
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"$K" --csv \
    python tools/prof_workload.py $W 3 2>/dev/null | grep -E "gpu__time_duration" | awk -F'","' '{print $NF}' | tr -d '"'
