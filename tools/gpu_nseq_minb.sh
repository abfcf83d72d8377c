cd $GRAFT_REPO_ROOT
run() { env $2 timeout 120 python bench.py --n-seq $1 --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/k.json 2>gpurun_out/k.log
  python -c "import json;d=json.load(open('gpurun_out/k.json'));print('nseq $1 $2', 'ms/step %.3f'%d['ms_per_step'], {k:round(v,3) for k,v in d['stages_ms'].items()})" 2>/dev/null || grep -m2 -i error gpurun_out/k.log; }
run 32 ME_PA_MINB=4; run 32 ME_PA_MINB=1; run 32 ME_PA_MINB=2
run 64 ME_PA_MODE=hybrid; run 64 ME_PA_MODE=duo-hybrid; run 96 ME_PA_MINB=4; run 96 ME_PA_MODE=hybrid
run 128 ME_PA_MODE=fast
