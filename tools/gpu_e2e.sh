cd $GRAFT_REPO_ROOT
timeout 180 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 100 -x 2>&1 | tail -2
timeout 300 python bench.py --steps 50 --warmup 3 --no-cpu > gpurun_out/e.json 2>gpurun_out/e.log
python -c "import json;d=json.load(open('gpurun_out/e.json'));print('ms/step %.3f'%d['ms_per_step'], {k:round(v,3) for k,v in d['stages_ms'].items()}, 'e2e', d['e2e'], 'clk', d['clocks'])" || tail -3 gpurun_out/e.log
