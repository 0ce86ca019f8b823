#!/bin/bash
# ncu launch lists of bench.py (gpu__time_duration per launch; shares of the step), summarised by
# tools/launch_summary.py into gpurun_out/launches_summary.md
mkdir -p gpurun_out
A="--steps 2 --warmup 3 --no-e2e --no-configs --no-cpu-baseline --no-dropin"
B="--steps 1 --warmup 3 --no-e2e --no-probe --no-cpu-baseline --no-dropin"
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches.csv python bench.py $A > gpurun_out/launches_a.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_configs.csv python bench.py $B > gpurun_out/launches_b.log 2>&1
python tools/launch_summary.py gpurun_out/launches_summary.md \
  "bench.py $A (the timed region: 5 launches of the headline kernel)=gpurun_out/launches.csv" \
  "bench.py $B (headline + cfg1..cfg4 + few-long-messages points)=gpurun_out/launches_configs.csv"
