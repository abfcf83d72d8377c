cd $GRAFT_REPO_ROOT
export ME_PA_KEY_A=1 ME_PA_KEY_S=0
for v in "0 64" "1 64" "0 16" "1 16" "1 256"; do
  set -- $v
  for wl in cfg2-pa cfg4-pa; do
  ME_PA_STATIC=$1 ME_PA_POLL_NS=$2 timeout 120 python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/v.json 2>gpurun_out/v.log
  python -c "import json;d=json.load(open('gpurun_out/v.json'));print('$wl static=$1 poll=$2', 'ms/step %.3f'%d['ms_per_step'], 'search %.3f'%d['stages_ms']['search'])" || tail -3 gpurun_out/v.log
  done
done
