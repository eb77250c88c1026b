# On the GPU box: render FPS with 2 and 3 frame-stream buffer sets.
for i in 1 2; do
for n in 2 3; do
timeout 300 python -c "
import sys; sys.argv=['bench.py','--steps','20','--warmup','5','--no-cpu-baseline']
import paper_2411_19588_b200.engine as e; e.StepEngine.RENDER_SETS=$n
import bench; bench.main()" > gpurun_out/sets_$n.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/sets_$n.log').read().strip().splitlines()[-1]); print($n, d['ms_per_step'], {k: v['fps'] for k, v in d['render_fps'].items()})"
done; done
