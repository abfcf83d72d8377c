# Dependency-poll interval sweep on the cfg4 search stage.
cd $GRAFT_REPO_ROOT
for ns in 0 32 64 128 256; do
  ME_PA_POLL_NS=$ns timeout 120 python bench.py --steps 30 --warmup 3 --no-cpu --no-e2e > gpurun_out/k.json 2>gpurun_out/k.log
  python -c "import json;d=json.load(open('gpurun_out/k.json'));print('poll_ns $ns', 'ms/step %.4f'%d['ms_per_step'], 'search %.4f'%d['stages_ms']['search'])" || tail -3 gpurun_out/k.log
done
