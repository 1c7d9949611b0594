cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_cache.py tests/test_gpu_verify.py -x -q -p no:cacheprovider 2>&1 | tail -30
