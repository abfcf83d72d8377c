cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/sched
timeout 900 python tools/key_probe.py 256,32 default bytes:pa_byte_masks=1 > gpurun_out/sched/bits.txt 2>&1; echo rc=$?
cat gpurun_out/sched/bits.txt

