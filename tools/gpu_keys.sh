cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 -x 2>&1 | tail -3
for ks in "1 1" "1 0" "2 1" "3 1" "4 1" "1 2"; do
  set -- $ks
  ME_PA_KEY_A=$1 ME_PA_KEY_S=$2 timeout 300 python bench.py --steps 30 --warmup 3 --no-cpu --no-e2e > gpurun_out/k.json 2>/dev/null
  python -c "import json;d=json.load(open('gpurun_out/k.json'));print('A=$1 S=$2', 'ms/step %.3f'%d['ms_per_step'], {k:round(v,3) for k,v in d['stages_ms'].items()})"
done
