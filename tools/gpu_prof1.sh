cd $GRAFT_REPO_ROOT
NCU=/usr/local/cuda/bin/ncu
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches_cfg4.csv python tools/profile_solve.py --config cfg4 > gpurun_out/prof_run1.log 2>&1
echo launches rc=$?
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_dense_linearize -s 2 -c 1 -o gpurun_out/prof_lin python tools/profile_solve.py --config cfg4 > gpurun_out/prof_run2.log 2>&1
echo lin rc=$?
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_pcg -s 2 -c 1 -o gpurun_out/prof_pcg python tools/profile_solve.py --config cfg4 > gpurun_out/prof_run3.log 2>&1
echo pcg rc=$?
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_overlap -c 1 -o gpurun_out/prof_overlap python tools/profile_solve.py --config cfg4 --max-iterations 1 > gpurun_out/prof_run4.log 2>&1
echo overlap rc=$?
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:k_dense_energy -s 2 -c 1 -o gpurun_out/prof_energy python tools/profile_solve.py --config cfg4 > gpurun_out/prof_run5.log 2>&1
echo energy rc=$?
