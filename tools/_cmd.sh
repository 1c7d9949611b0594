cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/pytest_gpu.log
for v in trace; do echo == $v; SFB_LIB=$GRAFT_REPO_ROOT/variants/$v.so timeout 300 python tools/pcg_trace.py; done
VARIANTS="cur" bash tools/gpu_variants.sh
