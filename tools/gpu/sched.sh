cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sched
timeout 900 python tools/seq_schedule_probe.py 2 3 5 > gpurun_out/sched/spec.txt 2>&1
timeout 900 python tools/key_probe.py 256,32 default >> gpurun_out/sched/spec.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/sched/pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/sched/pytest.log
cat gpurun_out/sched/spec.txt
