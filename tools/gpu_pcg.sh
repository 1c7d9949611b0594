cd $GRAFT_REPO_ROOT
for b in 0 32 128; do echo "== blocks $b"; SFB_PCG_BLOCKS=$b timeout 300 python tools/pcg_bench.py; done > gpurun_out/pcg_bench.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_reference_suite.py -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
echo done
