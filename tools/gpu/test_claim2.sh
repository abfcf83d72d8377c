cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/t4
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x --timeout 300 > gpurun_out/t4/pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/t4/pytest.log
for c in 1 0 1 0; do
ME_PA_CLAIM=$c timeout 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu --no-es --no-parity > gpurun_out/t4/b$c.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/t4/b$c.json'));print('claim=$c', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['stages_ms'].items()})"
done
for n in 1 16; do
for c in 1 0; do
ME_PA_CLAIM=$c timeout 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu --no-es --no-parity --n-seq $n > gpurun_out/t4/n$n$c.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/t4/n$n$c.json'));print('n=$n claim=$c', round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['stages_ms'].items()})"
done; done
