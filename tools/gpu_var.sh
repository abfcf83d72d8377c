cd $GRAFT_REPO_ROOT
for v in 64 256 1000; do
  ME_PA_POLL_NS=$v timeout 120 python bench.py --steps 30 --warmup 3 --no-cpu --no-e2e > gpurun_out/v.json 2>gpurun_out/v.log
  python -c "import json;d=json.load(open('gpurun_out/v.json'));print('poll=$v', 'ms/step %.3f'%d['ms_per_step'], 'search %.3f'%d['stages_ms']['search'])" || tail -3 gpurun_out/v.log
done
for ks in "1 0" "4 1" "8 1"; do
  set -- $ks
  ME_PA_KEY_A=$1 ME_PA_KEY_S=$2 timeout 120 python bench.py --steps 30 --warmup 3 --no-cpu --no-e2e > gpurun_out/v.json 2>gpurun_out/v.log
  python -c "import json;d=json.load(open('gpurun_out/v.json'));print('key $1 $2', 'ms/step %.3f'%d['ms_per_step'], 'search %.3f'%d['stages_ms']['search'])" || tail -3 gpurun_out/v.log
done
