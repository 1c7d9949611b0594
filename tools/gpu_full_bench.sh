cd $GRAFT_REPO_ROOT
( time timeout 1500 python bench.py > gpurun_out/bench_full.log 2> gpurun_out/bench_full.err ) 2> gpurun_out/bench_full.time
echo bench rc=$?
( time timeout 1500 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2> gpurun_out/bench_ref.err ) 2> gpurun_out/bench_ref.time
echo ref rc=$?
