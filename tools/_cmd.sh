cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_suite.py tests/test_gpu_fullsize.py -x -q -p no:cacheprovider 2>&1 | tail -2
VARIANTS="cur" bash tools/gpu_variants.sh
