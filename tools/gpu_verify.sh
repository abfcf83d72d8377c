# Round-end rehearsal: full GPU suite, smoke, default bench line.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/v
timeout 1500 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/v/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -n 5 gpurun_out/v/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/v/smoke.log 2>&1; echo smoke rc=$?; tail -n 2 gpurun_out/v/smoke.log
timeout 600 python bench.py > gpurun_out/v/bench.json 2> gpurun_out/v/bench.log; echo bench rc=$?
python -c "import json;d=json.load(open('gpurun_out/v/bench.json'));print(d['ms_per_step'], d['value'], d['stages_ms'], d['e2e']['value'], d['clocks'])"
