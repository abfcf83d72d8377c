cd $GRAFT_REPO_ROOT
timeout 180 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 100 -x 2>&1 | tail -15
for mode in group warp; do
for wl in cfg4-pa cfg2-pa; do
  ME_PA_MODE=$mode ME_PA_KEY_A=1 ME_PA_KEY_S=0 timeout 120 python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/k.json 2>gpurun_out/k.log
  python -c "import json;d=json.load(open('gpurun_out/k.json'));print('$mode $wl', 'ms/step %.3f'%d['ms_per_step'], {k:round(v,3) for k,v in d['stages_ms'].items()})" || tail -3 gpurun_out/k.log
done
done
