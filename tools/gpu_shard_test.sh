cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo pytest rc=$?
