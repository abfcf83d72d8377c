cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/spec
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/spec/pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/spec/pytest.log
timeout 600 python tools/key_probe.py 16,32,64,256 default nospec:pa_no_spec=1 > gpurun_out/spec/probe.txt 2>&1; echo probe rc=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-es --no-bits --no-parity > gpurun_out/spec/bench.json 2> gpurun_out/spec/bench.log; echo bench rc=$?
