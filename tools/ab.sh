#!/bin/bash
# On the GPU box: time bench.py with each library variant in build/variants (plus the in-tree one as "base").
# usage: tools/ab.sh [steps]
steps=${1:-20}
lib=paper_2411_19588_b200/libuwsplat_b200.so
cp $lib /tmp/base.so
for v in base build/variants/*.so; do
  name=$(basename $v .so)
  if [ "$v" = base ]; then cp /tmp/base.so $lib; else cp $v $lib; fi
  timeout 300 python bench.py --steps $steps --warmup 5 --no-cpu-baseline --no-render-fps > gpurun_out/ab_$name.log 2>&1
  python - "$name" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}.log").read().strip().splitlines()[-1])
st = d["stages_ms"]
print(sys.argv[1], d["ms_per_step"], {k.replace("uws_", ""): v for k, v in st.items()})
PY
done
cp /tmp/base.so $lib
