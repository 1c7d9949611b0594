# Parity tests + a device-only bench line (+ optional e2e breakdown): the inner loop.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo pytest rc=$?; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline ${BENCH_EXTRA:-} > gpurun_out/bench.log 2>&1
echo bench rc=$?; tail -1 gpurun_out/bench.log | cut -c1-1500
if [ -n "$E2E" ]; then timeout 600 python tools/e2e_breakdown.py cfg4 > gpurun_out/e2e.log 2>&1; echo e2e rc=$?; cat gpurun_out/e2e.log | tail -5; fi
