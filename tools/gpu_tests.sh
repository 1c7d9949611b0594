# GPU tests only (optionally a subset: TESTS="tests/test_x.py ..."), log under gpurun_out/.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout ${TEST_TIMEOUT:-1500} python -m pytest ${TESTS:-tests} -x -q -m gpu -p no:cacheprovider ${PYTEST_EXTRA:-} > gpurun_out/pytest_gpu.log 2>&1
echo pytest rc=$?; tail -15 gpurun_out/pytest_gpu.log
