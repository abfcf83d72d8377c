# usage: gpu_env.sh "ENV1=a ENV2=b" "ENV1=c" ...   (cfg4-pa search-stage timing per env set)
cd $GRAFT_REPO_ROOT
timeout 180 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q --timeout 100 -x 2>&1 | tail -1
for envs in "$@"; do
  env $envs timeout 120 python bench.py --workload ${WL:-cfg4-pa} --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/k.json 2>gpurun_out/k.log
  python -c "import json;d=json.load(open('gpurun_out/k.json'));print('$envs', 'ms/step %.3f'%d['ms_per_step'], {k:round(v,3) for k,v in d['stages_ms'].items()})" || tail -3 gpurun_out/k.log
done
