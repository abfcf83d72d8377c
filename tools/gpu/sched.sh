cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sched
timeout 900 python tools/key_probe.py 256,128 default alias:pa_poll_ns=63 > gpurun_out/sched/alias.txt 2>&1; echo rc=$?
cat gpurun_out/sched/alias.txt
