cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_suite.py -x -q -p no:cacheprovider 2>&1 | tail -2
for v in trace; do echo == $v; SFB_LIB=$GRAFT_REPO_ROOT/variants/$v.so timeout 300 python tools/pcg_trace.py; done
VARIANTS="cur" bash tools/gpu_variants.sh
