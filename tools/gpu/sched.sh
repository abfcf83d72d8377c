cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sched
timeout 900 python tools/key_probe.py 16,32,64,128 default fast1:pa_schedule=2,pa_fast_ctas=1 fast2:pa_schedule=2,pa_fast_ctas=2 fast3:pa_schedule=2,pa_fast_ctas=3 fast4:pa_schedule=2,pa_fast_ctas=4 quad:pa_schedule=5 quadw20:pa_schedule=5,pa_wide_blocks=2960 quadw10:pa_schedule=5,pa_wide_blocks=1480 > gpurun_out/sched/probe.txt 2>&1; echo probe rc=$?
