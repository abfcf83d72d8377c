cd $GRAFT_REPO_ROOT
for wl in cfg2-pa cfg3-pa cfg5-pa; do
for m in duo fast warp; do
  ME_PA_MODE=$m timeout 600 python bench.py --workload $wl --frames 6 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/m.json 2>gpurun_out/m.log
  python -c "import json;d=json.load(open('gpurun_out/m.json'));print('$wl $m', 'ms %.3f'%d['ms_per_step'], {k:round(v,3) for k,v in d['stages_ms'].items()})" || tail -2 gpurun_out/m.log
done; done
