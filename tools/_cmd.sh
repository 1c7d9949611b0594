cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
for c in cfg4 cfg5; do SFB_TRACE=1 timeout 300 python tools/profile_solve.py --config $c --solves 3 2>&1 | grep 'rebuild_structure' | tail -1; done
CFG=cfg5 VARIANTS="cur" bash tools/gpu_variants.sh
