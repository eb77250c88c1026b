for i in 1 2; do
python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c4_on.log 2>&1
python -c "
import sys; sys.argv=['bench.py','--config','c4','--steps','3','--warmup','3','--no-cpu-baseline']
import paper_2411_19588_b200.engine as e; e.StepEngine.OVERLAP_VIEWS=False
import bench; bench.main()" > gpurun_out/c4_off.log 2>&1
for v in on off; do python -c "
import json; d=json.loads(open('gpurun_out/c4_$v.log').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'])"; done
done
