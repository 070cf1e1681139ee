#!/bin/bash
# Run on the GPU box (gpurun): launch list of the bench's timed region and one
# `ncu --set full` capture per hot kernel family, exported to CSV on the box
# (reports are too large to bring back).  Outputs in gpurun_out/.
set -u
OUT=gpurun_out
P=tools/prof_workload.py
python bench.py --steps 5 --warmup 3 --no-extras --no-cpu --no-sustain > $OUT/bench_plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-extras --no-cpu --no-sustain > $OUT/ncu_launch.log 2>&1
for w in ${WORKLOADS:-pool16 conv3 conv5 conv7 conv1d nchw pool64 pool255}; do
  timeout 120 python $P $w 1 > $OUT/plain_$w.log 2>&1 &&
  timeout 900 ncu -f --set full --clock-control none --import-source on \
      -k regex:"pool_|conv2d_|nchw|tc_" -c ${NCU_COUNT:-3} -o /tmp/prof_$w python $P $w 1 > $OUT/ncu_$w.log 2>&1
  if [ -f /tmp/prof_$w.ncu-rep ]; then
    ncu -i /tmp/prof_$w.ncu-rep --page raw --csv > $OUT/raw_$w.csv 2>/dev/null
    ncu -i /tmp/prof_$w.ncu-rep --page details --csv > $OUT/details_$w.csv 2>/dev/null
    ncu -i /tmp/prof_$w.ncu-rep --page source --csv --print-source sass > $OUT/source_$w.csv 2>/dev/null
    gzip -f $OUT/source_$w.csv
  fi
done
ls -la $OUT
