cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
SFB_TRACE=1 timeout 300 python tools/profile_solve.py --config cfg4 --solves 3 2>&1 | grep rebuild | tail -2
VARIANTS="cur" bash tools/gpu_variants.sh
