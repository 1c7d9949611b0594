cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider 2>&1 | tail -2
for c in cfg4 cfg5; do echo == $c; timeout 600 python tools/e2e_breakdown.py $c 2>&1 | grep rep | tail -2; done
