cd $GRAFT_REPO_ROOT
for ns in 8 32 64 128 256; do
for m in duo fast; do
  ME_PA_MODE=$m timeout 600 python bench.py --workload cfg4-pa --n-seq $ns --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/m.json 2>gpurun_out/m.log
  python -c "import json;d=json.load(open('gpurun_out/m.json'));print('nseq $ns $m', 'search %.3f'%d['stages_ms']['search'])" || tail -2 gpurun_out/m.log
done; done
