# Ring-search baselines (configs 3 and 5) and the ES line: device-side numbers.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/rings
for wl in cfg3-tss cfg3-fss cfg3-ds cfg5-tss cfg5-fss cfg5-ds cfg3-pa; do
  timeout 300 python bench.py --workload $wl --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/rings/$wl.json 2> gpurun_out/rings/$wl.log
  python -c "import json;d=json.load(open('gpurun_out/rings/$wl.json'));print('$wl', 'ms/step %.3f'%d['ms_per_step'], 'MB/s %.3g'%d['value'], {k:round(v,3) for k,v in d['stages_ms'].items()}, 'frac', round(d['roofline']['frac'],3))" || tail -3 gpurun_out/rings/$wl.log
done
