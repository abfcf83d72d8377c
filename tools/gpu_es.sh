cd $GRAFT_REPO_ROOT
./tools/int_peak > gpurun_out/int_peak.json; cat gpurun_out/int_peak.json
mkdir -p profiles; cp gpurun_out/int_peak.json profiles/int_peak.json
timeout 600 python bench.py --workload cfg5-es --frames 6 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/es5.json 2>gpurun_out/es5.log
python -c "import json;d=json.load(open('gpurun_out/es5.json'));print('cfg5-es ms/step %.3f'%d['ms_per_step'], d['stages_ms'], d['roofline'])" || tail -3 gpurun_out/es5.log
timeout 600 python bench.py --workload cfg2-es --steps 10 --warmup 3 --no-cpu --no-e2e > gpurun_out/es2.json 2>gpurun_out/es2.log
python -c "import json;d=json.load(open('gpurun_out/es2.json'));print('cfg2-es ms/step %.3f'%d['ms_per_step'], d['stages_ms'], d['roofline'])" || tail -3 gpurun_out/es2.log
for w in cfg3-tss cfg3-fss cfg3-ds; do
timeout 600 python bench.py --workload $w --frames 6 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/r.json 2>gpurun_out/r.log
python -c "import json;d=json.load(open('gpurun_out/r.json'));print('$w ms/step %.3f'%d['ms_per_step'], d['stages_ms'])" || tail -3 gpurun_out/r.log
done
