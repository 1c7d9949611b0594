# Full round check on one B200: smoke, GPU parity tests, bench (ours + reference arm),
# row benches, ncu launch list and --set full captures of the top kernels.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo smoke rc=$?
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo pytest rc=$?
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1
echo bench rc=$?
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
echo benchref rc=$?
timeout 600 python tools/bench_verify.py --config cfg4 > gpurun_out/bench_verify.log 2>&1
echo verify rc=$?
timeout 600 python tools/bench_cache.py > gpurun_out/bench_cache.log 2>&1
echo cache rc=$?
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv python tools/profile_solve.py --config cfg4 --solves 2 > gpurun_out/launch_run.log 2>&1
echo launches rc=$?
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_dense_fused -s 3 -c 1 -o gpurun_out/prof_fused python tools/profile_solve.py --config cfg4 > gpurun_out/prof_fused.log 2>&1
echo prof rc=$?
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_pcg -s 2 -c 1 -o gpurun_out/prof_pcg python tools/profile_solve.py --config cfg4 > gpurun_out/prof_pcg.log 2>&1
echo profpcg rc=$?
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_dense_verify -c 1 -o gpurun_out/prof_verify python tools/bench_verify.py --config cfg4 --reps 1 --cpu-sample 2 > gpurun_out/prof_verify.log 2>&1
echo profverify rc=$?
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_cache_reduce -c 1 -o gpurun_out/prof_cache python tools/bench_cache.py --frames 64 --reps 1 > gpurun_out/prof_cache.log 2>&1
echo profcache rc=$?
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launch_bench_run.log 2>&1
echo launchbench rc=$?
timeout 600 python tools/bench_tsdf.py > gpurun_out/bench_tsdf.log 2>&1
echo tsdf rc=$?
for c in cfg3 cfg5; do timeout 900 python bench.py --config $c > gpurun_out/bench_$c.log 2>&1; echo bench$c rc=$?; done
