# Inner loop: variant timings (VARIANTS, default "cur") then parity tests (TESTS, default all -m gpu)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
VARIANTS=${VARIANTS:-cur} bash tools/gpu_variants.sh 2>&1 | tee gpurun_out/variants.log
timeout ${TEST_TIMEOUT:-1500} python -m pytest ${TESTS:-tests} -x -q -m gpu -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo pytest rc=$?; tail -15 gpurun_out/pytest_gpu.log
