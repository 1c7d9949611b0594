# One ncu --set full capture (with source) of the 4th k_dense_fused launch at cfg4
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
TAG=${TAG:-dense}
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:${KREGEX:-k_dense_fused} -s ${SKIP:-3} -c 1 -o gpurun_out/prof_$TAG python tools/profile_solve.py --config ${CFG:-cfg4} > gpurun_out/prof_$TAG.log 2>&1
echo prof rc=$?; tail -3 gpurun_out/prof_$TAG.log
ls -la gpurun_out/
