cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sched
timeout 300 python tools/key_probe.py 8 default df:pa_dataflow=1 > gpurun_out/sched/df.txt 2>&1; echo rc=$?
timeout 600 python tools/key_probe.py 32,64,256 default df:pa_dataflow=1 df3:pa_dataflow=1,pa_fast_ctas=3 df2:pa_dataflow=1,pa_fast_ctas=2 >> gpurun_out/sched/df.txt 2>&1; echo rc=$?
cat gpurun_out/sched/df.txt
