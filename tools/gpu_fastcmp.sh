cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q --timeout 200 -x 2>&1 | tail -1
for wl in cfg2-pa cfg3-pa cfg5-pa; do
  timeout 600 python bench.py --workload $wl --frames 6 --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/m.json 2>gpurun_out/m.log
  python -c "import json;d=json.load(open('gpurun_out/m.json'));print('$wl', 'ms %.3f'%d['ms_per_step'], 'search %.3f'%d['stages_ms']['search'])" || tail -2 gpurun_out/m.log
done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e > gpurun_out/m.json 2>gpurun_out/m.log
python -c "import json;d=json.load(open('gpurun_out/m.json'));print('cfg4', 'ms %.3f'%d['ms_per_step'], {k:round(v,3) for k,v in d['stages_ms'].items()})"
