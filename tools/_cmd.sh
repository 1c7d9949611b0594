cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
VARIANTS="cur mb1 mb3" bash tools/gpu_variants.sh
timeout 300 python tools/e2e_breakdown.py cfg4 2>&1 | tail -4
