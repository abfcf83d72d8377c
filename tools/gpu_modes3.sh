cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q --timeout 200 -x 2>&1 | tail -1
for wl in cfg2-pa cfg3-pa cfg5-pa; do
for mb in 4 5 3; do
  ME_PA_MINB=$mb timeout 600 python bench.py --workload $wl --frames 6 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/m.json 2>gpurun_out/m.log
  python -c "import json;d=json.load(open('gpurun_out/m.json'));print('$wl minb $mb', 'search %.3f'%d['stages_ms']['search'])" || tail -2 gpurun_out/m.log
done; done
