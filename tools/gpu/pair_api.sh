cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pp
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/pp/launches.csv python tools/pair_api_probe.py 1 12 > gpurun_out/pp/ncu.log 2>&1; echo rc=$?
python tools/launch_summary.py gpurun_out/pp/launches.csv 2>&1 | head -20
