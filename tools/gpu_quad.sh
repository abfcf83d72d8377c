cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 100 -x -k "modes" 2>&1 | tail -3
for envs in "ME_PA_MODE=hybrid" "ME_PA_MODE=quad" "ME_PA_MODE=quad ME_PA_QMINB=3" "ME_PA_MODE=quad ME_PA_QMINB=2"; do
  env $envs timeout 120 python bench.py --workload ${WL:-cfg4-pa} --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/k.json 2>gpurun_out/k.log
  python -c "import json;d=json.load(open('gpurun_out/k.json'));print('$envs', 'ms/step %.3f'%d['ms_per_step'], {k:round(v,3) for k,v in d['stages_ms'].items()})" || tail -3 gpurun_out/k.log
done
