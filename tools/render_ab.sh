#!/bin/bash
# On the GPU box: render FPS (bench's frame stream) with each library variant in build/variants.
lib=paper_2411_19588_b200/libuwsplat_b200.so
cp $lib /tmp/base.so
for v in base build/variants/*.so; do
  name=$(basename $v .so)
  if [ "$v" = base ]; then cp /tmp/base.so $lib; else cp $v $lib; fi
  python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/rab_$name.log 2>&1
  python - "$name" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/rab_{sys.argv[1]}.log").read().strip().splitlines()[-1])
print(sys.argv[1], d["ms_per_step"], d["render_fps"])
PY
done
cp /tmp/base.so $lib
