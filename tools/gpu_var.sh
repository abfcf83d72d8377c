cd $GRAFT_REPO_ROOT
export ME_PA_KEY_A=1 ME_PA_KEY_S=0
timeout 180 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 100 -x 2>&1 | tail -2
for v in "group 64" "group 300" "group 1000" "warp 300"; do
  set -- $v
  for wl in cfg2-pa cfg4-pa; do
  ME_PA_MODE=$1 ME_PA_POLL_NS=$2 timeout 120 python bench.py --workload $wl --steps 20 --warmup 3 --no-cpu --no-e2e > gpurun_out/v.json 2>gpurun_out/v.log
  python -c "import json;d=json.load(open('gpurun_out/v.json'));print('$wl $1 poll=$2', 'ms/step %.3f'%d['ms_per_step'], 'search %.3f'%d['stages_ms']['search'])" || tail -3 gpurun_out/v.log
  done
done
