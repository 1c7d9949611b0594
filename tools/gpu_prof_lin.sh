cd $GRAFT_REPO_ROOT
timeout 900 /usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:k_dense_fused -s 3 -c 1 -o gpurun_out/prof_fused python tools/profile_solve.py --config cfg4 > gpurun_out/prof_fused.log 2>&1
echo rc=$?
