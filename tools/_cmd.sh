cd $GRAFT_REPO_ROOT
VARIANTS="cur epf" bash tools/gpu_variants.sh
