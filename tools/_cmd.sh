cd $GRAFT_REPO_ROOT
ls variants/
SFB_LIB=$GRAFT_REPO_ROOT/variants/dmma3.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -3
VARIANTS="cur dmma2 dmma3" bash tools/gpu_variants.sh
