cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sched
timeout 900 python tools/key_probe.py 32,48,64 default h15:pa_schedule=5,pa_wide_blocks=1500 h25:pa_schedule=5,pa_wide_blocks=2500 h35:pa_schedule=5,pa_wide_blocks=3500 h25f3:pa_schedule=5,pa_wide_blocks=2500,pa_fast_ctas=3 q2h25:pa_schedule=5,pa_wide_blocks=2500,pa_quad_ctas=2 > gpurun_out/sched/mid.txt 2>&1; echo rc=$?
cat gpurun_out/sched/mid.txt
