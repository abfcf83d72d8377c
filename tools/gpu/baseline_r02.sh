cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/b0
timeout 600 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/b0/pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/b0/pytest.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/b0/bench.json 2> gpurun_out/b0/bench.log; echo bench rc=$?
python -c "import json;d=json.load(open('gpurun_out/b0/bench.json'));print(d['ms_per_step'], d['stages_ms'], d['clocks'])"
nproc; lscpu | grep -i 'model name\|^CPU(s)\|Thread'
