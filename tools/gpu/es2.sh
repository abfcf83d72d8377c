cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x --timeout 300 -k "es or ES or block_search or sequence or big or golden or band" > /tmp/p.log 2>&1; echo pytest rc=$?; tail -2 /tmp/p.log
timeout 600 python bench.py --workload cfg5-es --es-steps 10 --no-parity > /tmp/es.json 2>/tmp/es.log; echo rc=$?
python -c "import json;d=json.load(open('/tmp/es.json'));print(d['ms_per_step'], d['roofline']['frac'], d['roofline']['achieved'], d['roofline']['peak'], d['clocks'])"
