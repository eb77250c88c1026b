#!/bin/bash
# On the GPU box: ncu launch list (per-kernel durations) of a short bench run.
# usage: tools/launchlist.sh TAG [extra bench args]
tag=$1; shift
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches_$tag.csv python bench.py --steps 3 --warmup 3 \
  --no-cpu-baseline --no-render-fps "$@" > gpurun_out/ncu_$tag.log 2>&1
python tools/launches.py gpurun_out/launches_$tag.csv 40 > gpurun_out/launches_${tag}_summary.txt
