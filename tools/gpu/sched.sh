cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sched
timeout 900 python tools/key_probe.py 256,128,64 default q5:pa_quad_ctas=5 q4:pa_quad_ctas=4 > gpurun_out/sched/slots.txt 2>&1; echo rc=$?
cat gpurun_out/sched/slots.txt
