# One line per workload (device value + stages), small step counts.
cd $GRAFT_REPO_ROOT
for wl in cfg1-pa cfg2-pa cfg2-es cfg3-pa cfg3-tss cfg3-fss cfg3-ds cfg5-pa cfg5-es cfg5-tss; do
  case $wl in cfg3-*|cfg5-*) extra="--frames 6 --steps 3";; *) extra="--steps 20";; esac
  timeout 600 python bench.py --workload $wl $extra --warmup 3 --no-cpu --no-e2e > gpurun_out/wl_$wl.json 2>gpurun_out/wl_$wl.log
  python -c "import json;d=json.load(open('gpurun_out/wl_$wl.json'));r=d.get('roofline') or {};print('$wl', 'value %.4g'%d['value'], 'ms %.3f'%d['ms_per_step'], {k:round(v,3) for k,v in d['stages_ms'].items()}, 'frac', r.get('frac'))" || tail -2 gpurun_out/wl_$wl.log
done
