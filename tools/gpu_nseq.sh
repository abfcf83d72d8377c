cd $GRAFT_REPO_ROOT
for ns in 32 64 128 256 512; do
  timeout 120 python bench.py --workload cfg4-pa --n-seq $ns --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/k.json 2>gpurun_out/k.log
  python -c "import json;d=json.load(open('gpurun_out/k.json'));print('nseq $ns', 'ms/step %.3f'%d['ms_per_step'], {k:round(v,3) for k,v in d['stages_ms'].items()})" || tail -3 gpurun_out/k.log
done
