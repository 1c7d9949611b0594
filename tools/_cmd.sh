cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
CFG=cfg5 VARIANTS="cur" bash tools/gpu_variants.sh
VARIANTS="cur" bash tools/gpu_variants.sh
