# GPU test pass used during development: headline parity first, then the rest
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests/test_gpu_headline.py -q --tb=short -p no:cacheprovider ${HEADLINE_ARGS} > gpurun_out/headline.log 2>&1
echo "headline rc=$?" >> gpurun_out/headline.log
timeout 1200 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider --deselect tests/test_gpu_headline.py > gpurun_out/gpu_all.log 2>&1
echo "all rc=$?" >> gpurun_out/gpu_all.log
