cd $GRAFT_REPO_ROOT
timeout 180 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 -x 2>&1 | tail -15
for ks in "1 0" "2 1"; do
  set -- $ks
  ME_PA_KEY_A=$1 ME_PA_KEY_S=$2 timeout 120 python bench.py --steps 30 --warmup 3 --no-cpu --no-e2e > gpurun_out/k.json 2>gpurun_out/k.log
  python -c "import json;d=json.load(open('gpurun_out/k.json'));print('A=$1 S=$2', 'ms/step %.3f'%d['ms_per_step'], {k:round(v,3) for k,v in d['stages_ms'].items()})" || tail -5 gpurun_out/k.log
done
ME_PA_KEY_A=1 ME_PA_KEY_S=0 timeout 120 python bench.py --workload cfg2-pa --steps 30 --warmup 3 --no-cpu --no-e2e > gpurun_out/k2.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/k2.json'));print('cfg2-pa', 'ms/step %.3f'%d['ms_per_step'], {k:round(v,3) for k,v in d['stages_ms'].items()})"
ME_PA_KEY_A=1 ME_PA_KEY_S=0 ME_PA_TRACE=gpurun_out/trace_cfg2.bin timeout 120 python bench.py --workload cfg2-pa --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>gpurun_out/t.log
ME_PA_KEY_A=1 ME_PA_KEY_S=0 ME_PA_TRACE=gpurun_out/trace_cfg4.bin timeout 120 python bench.py --workload cfg4-pa --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>gpurun_out/t4.log
