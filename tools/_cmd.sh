cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_tsdf.py -x -q -p no:cacheprovider 2>&1 | tail -30
