# Full round check on one B200: smoke, GPU parity tests, bench (ours + reference arm),
# ncu launch list and one --set full capture of the dense pass.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo smoke rc=$?
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo pytest rc=$?
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1
echo bench rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
echo benchref rc=$?
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv python tools/profile_solve.py --config cfg4 --solves 2 > gpurun_out/launch_run.log 2>&1
echo launches rc=$?
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_dense_fused -s 3 -c 1 -o gpurun_out/prof_fused python tools/profile_solve.py --config cfg4 > gpurun_out/prof_fused.log 2>&1
echo prof rc=$?
