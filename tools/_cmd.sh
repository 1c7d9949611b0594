cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_verify.py tests/test_gpu_cache.py -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 600 python tools/bench_verify.py --config cfg4 2>&1 | tail -1
