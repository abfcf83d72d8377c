cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/full
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/full/pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/full/pytest.log
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/full/bench.json 2> gpurun_out/full/bench.log; echo bench rc=$?
python -c "import json;d=json.load(open('gpurun_out/full/bench.json'));print(round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['stages_ms'].items()}, d['parity']['mismatches'], d['es_cfg5']['roofline']['frac'], d['clocks']['samples'], d['e2e']['value'])"
