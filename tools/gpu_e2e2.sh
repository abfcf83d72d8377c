cd $GRAFT_REPO_ROOT
nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket" | head -5
for envs in "ME_B200_CHUNKS=8" "ME_B200_CHUNKS=16" "ME_B200_CHUNKS=32"; do
  env $envs timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --e2e-steps 5 > gpurun_out/e.json 2>gpurun_out/e.log
  python -c "import json;d=json.load(open('gpurun_out/e.json'));e=d['e2e'];print('$envs', 'e2e ms %.2f'%(e['s_per_step']*1e3), 'MB/s %.3g'%e['value'], 'h2d', e['h2d_bytes_per_step'], 'd2h', e['d2h_bytes_per_step'])" || tail -3 gpurun_out/e.log
done
