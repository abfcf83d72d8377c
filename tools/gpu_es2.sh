cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q --timeout 200 -x 2>&1 | tail -1
timeout 600 python bench.py --workload cfg5-es --frames 6 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/es5.json 2>gpurun_out/es5.log
python -c "import json;d=json.load(open('gpurun_out/es5.json'));r=d['roofline'];print('cfg5-es ms/step %.3f'%d['ms_per_step'], {k:round(v,3) for k,v in d['stages_ms'].items()}, 'frac %.3f'%r['frac'], 'ach %.2f'%r['achieved'])" || tail -3 gpurun_out/es5.log
timeout 600 python bench.py --workload cfg2-es --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/es2.json 2>gpurun_out/es2.log
python -c "import json;d=json.load(open('gpurun_out/es2.json'));r=d['roofline'];print('cfg2-es ms/step %.3f'%d['ms_per_step'], {k:round(v,3) for k,v in d['stages_ms'].items()}, 'frac %.3f'%r['frac'])" || tail -3 gpurun_out/es2.log
