# usage: gpu_sweep.sh "ENV1=a ENV2=b" ...   (cfg4-pa timing per env set, no tests)
cd $GRAFT_REPO_ROOT
for envs in "$@"; do
  env $envs timeout 120 python bench.py --workload ${WL:-cfg4-pa} --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/k.json 2>gpurun_out/k.log
  python -c "import json;d=json.load(open('gpurun_out/k.json'));print('$envs', 'ms/step %.3f'%d['ms_per_step'], {k:round(v,3) for k,v in d['stages_ms'].items()})" 2>/dev/null || grep -m2 -i "error" gpurun_out/k.log
done
