cd $GRAFT_REPO_ROOT
timeout 900 /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv python tools/profile_solve.py --config cfg4 --solves 2 > gpurun_out/launch_run.log 2>&1
echo rc=$?
