cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/key
timeout 600 python tools/key_probe.py 64,128,256 default plain:pa_key_plain=1 > gpurun_out/key/probe6.txt 2>&1; echo probe rc=$?
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/key/pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/key/pytest.log
