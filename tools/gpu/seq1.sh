cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s1
ME_PA_SEQ=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x --timeout 120 > gpurun_out/s1/pytest.log 2>&1; echo pytest rc=$?; tail -15 gpurun_out/s1/pytest.log
for n in 256 128 64; do
timeout 300 python bench.py --steps 20 --warmup 5 --n-seq $n --no-e2e --no-cpu > gpurun_out/s1/bench$n.json 2> gpurun_out/s1/bench$n.log; echo bench rc=$?
python -c "import json;d=json.load(open('gpurun_out/s1/bench$n.json'));print($n, d['ms_per_step'], d['stages_ms'])" || tail -5 gpurun_out/s1/bench$n.log
ME_PA_SEQ=0 timeout 300 python bench.py --steps 20 --warmup 5 --n-seq $n --no-e2e --no-cpu > gpurun_out/s1/bench0_$n.json 2> gpurun_out/s1/bench0_$n.log
python -c "import json;d=json.load(open('gpurun_out/s1/bench0_$n.json'));print('old', $n, d['ms_per_step'], d['stages_ms'])" || tail -5 gpurun_out/s1/bench0_$n.log
done
