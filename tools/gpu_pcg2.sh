cd $GRAFT_REPO_ROOT
for b in 0 16 32 48 96 148; do echo "== blocks $b"; SFB_PCG_BLOCKS=$b timeout 300 python tools/pcg_bench.py | tail -2; done > gpurun_out/pcg_bench.log 2>&1
