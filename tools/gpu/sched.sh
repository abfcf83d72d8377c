cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sched
timeout 900 python tools/key_probe.py 128,96,64,48,32,24,16,8 default f2:pa_fast_ctas=2 f3:pa_fast_ctas=3 f4:pa_fast_ctas=4 > gpurun_out/sched/fdef.txt 2>&1; echo rc=$?
cat gpurun_out/sched/fdef.txt
