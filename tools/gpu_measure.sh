# Measurement refresh: bench (cfg4 default, cfg3, cfg5), ncu launch list of the
# bench command, one --set full capture of k_dense_fused and of k_pcg_reg.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1
echo bench rc=$?; tail -1 gpurun_out/bench.log | cut -c1-300
for c in cfg3 cfg5; do timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_$c.log 2>&1; echo bench$c rc=$?; done
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/launch_bench_run.log 2>&1
echo launchbench rc=$?
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_dense_fused -s 3 -c 1 -o gpurun_out/prof_fused python tools/profile_solve.py --config cfg4 > gpurun_out/prof_fused.log 2>&1
echo prof rc=$?
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_pcg -s 2 -c 1 -o gpurun_out/prof_pcg python tools/profile_solve.py --config cfg4 > gpurun_out/prof_pcg.log 2>&1
echo profpcg rc=$?
