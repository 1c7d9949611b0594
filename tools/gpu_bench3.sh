# bench line (ours), the 2-rank gloo protocol run on one GPU, and the reference arm
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nproc; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python bench.py > gpurun_out/bench.log 2>&1
echo bench rc=$?; tail -1 gpurun_out/bench.log | cut -c1-600
timeout 900 python bench.py --gpus 2 --dist-backend gloo --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_gloo2.log 2>&1
echo gloo2 rc=$?; tail -1 gpurun_out/bench_gloo2.log | cut -c1-400
if [ -z "$NOREF" ]; then
timeout 1500 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref.log 2>&1
echo benchref rc=$?; tail -1 gpurun_out/bench_ref.log | cut -c1-1200
fi
