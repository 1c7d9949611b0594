cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo pytest rc=$?
timeout 600 python tools/e2e_breakdown.py cfg4 > gpurun_out/e2e.log 2>&1
echo e2e rc=$?
timeout 1200 python bench.py --config cfg4 --steps 3 --warmup 2 --no-cpu-baseline > gpurun_out/bench.log 2>&1
echo bench rc=$?
