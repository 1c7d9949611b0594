cd $GRAFT_REPO_ROOT
SFB_LIB=$GRAFT_REPO_ROOT/variants/frnd.so timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider 2>&1 | tail -1
VARIANTS="cur frnd" bash tools/gpu_variants.sh
