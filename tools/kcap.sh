#!/bin/bash
# On the GPU box: `ncu --set full` of the first launches of the kernels matching a regex in a
# short bench run; summary, raw CSV and source pages to gpurun_out/.
# usage: tools/kcap.sh TAG REGEX COUNT [bench args]
tag=$1; re=$2; cnt=$3; shift 3
ncu --set full --clock-control none --import-source on -k regex:"$re" -c $cnt -o /tmp/k_$tag \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-render-fps "$@" > gpurun_out/ncu_k_$tag.log 2>&1
python tools/ncu_summary.py /tmp/k_$tag.ncu-rep gpurun_out/k_${tag}_summary.txt gpurun_out/k_${tag}_traffic.json > /dev/null 2>&1
ncu -i /tmp/k_$tag.ncu-rep --page raw --csv > gpurun_out/k_${tag}_raw.csv 2>/dev/null
ncu -i /tmp/k_$tag.ncu-rep --page details --csv > gpurun_out/k_${tag}_details.csv 2>/dev/null
for k in $(ncu -i /tmp/k_$tag.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; i=h.index('Kernel Name')
seen=[]
for r in rows[2:]:
    n=r[i].split('(')[0].split('::')[-1].split('<')[0]
    if n not in seen: seen.append(n)
print(' '.join(seen))"); do
  ncu -i /tmp/k_$tag.ncu-rep --page source --csv -k regex:$k -c 1 > gpurun_out/k_${tag}_src_$k.csv 2>/dev/null
done
