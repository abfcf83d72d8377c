# PDL chaining of the hybrid's grids: parity, then cfg4 with and without.
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x --timeout 300 2>&1 | tail -2
for rep in 1 2; do for p in 1 0; do export ME_PDL_SORT=$p;
  ME_PA_PDL=$p timeout 120 python bench.py --steps 50 --warmup 3 --no-cpu --no-e2e > gpurun_out/k.json 2>gpurun_out/k.log
  python -c "import json;d=json.load(open('gpurun_out/k.json'));print('pdl $p', 'ms/step %.4f'%d['ms_per_step'], {k:round(v,4) for k,v in d['stages_ms'].items()})" || tail -3 gpurun_out/k.log
done; done
