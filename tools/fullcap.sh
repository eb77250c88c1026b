#!/bin/bash
# On the GPU box: one `ncu --set full` capture of the first step's kernels of a short bench run
# (after the same command ran clean without ncu). Report kept in /tmp (too large to bring back);
# the summary, the raw metric CSV and the source pages of the named kernels go to gpurun_out/.
# usage: tools/fullcap.sh TAG "kernel regex for source pages" [bench args]
tag=$1; shift
src=$1; shift
python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-render-fps "$@" > gpurun_out/plain_$tag.log 2>&1 && \
ncu --set full --clock-control none --import-source on -c 60 -o /tmp/full_$tag \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-render-fps "$@" > gpurun_out/ncu_full_$tag.log 2>&1
python tools/ncu_summary.py /tmp/full_$tag.ncu-rep gpurun_out/full_${tag}_summary.txt gpurun_out/full_${tag}_traffic.json > /dev/null 2>&1
ncu -i /tmp/full_$tag.ncu-rep --page raw --csv > gpurun_out/full_${tag}_raw.csv 2>/dev/null
for k in $src; do
  ncu -i /tmp/full_$tag.ncu-rep --page source --csv -k regex:$k -c 1 > gpurun_out/full_${tag}_src_$k.csv 2>/dev/null
done
ls -la gpurun_out/ /tmp/full_$tag.ncu-rep
