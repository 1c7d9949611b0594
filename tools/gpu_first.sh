set -x
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo smoke rc=$?
timeout 1200 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo pytest rc=$?
timeout 900 python bench.py --config cfg3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_cfg3.log 2>&1
echo bench3 rc=$?
timeout 1200 python bench.py --config cfg4 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/bench_cfg4.log 2>&1
echo bench4 rc=$?
