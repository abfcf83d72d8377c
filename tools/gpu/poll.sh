cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/poll
timeout 600 python tools/key_probe.py 1,8,32 default p0:pa_poll_ns=1 p16:pa_poll_ns=16 p32:pa_poll_ns=32 p128:pa_poll_ns=128 > gpurun_out/poll/probe.txt 2>&1; echo probe rc=$?
