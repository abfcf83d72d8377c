cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/f
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q -x --timeout 300 > gpurun_out/f/pytest.log 2>&1; echo pytest rc=$?; tail -3 gpurun_out/f/pytest.log
for i in 1 2; do
timeout 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu --no-es --no-parity > gpurun_out/f/b.json 2>/dev/null
python -c "import json;d=json.load(open('gpurun_out/f/b.json'));print(round(d['ms_per_step'],4), {k:round(v,4) for k,v in d['stages_ms'].items()})"
done
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-es --no-parity"
$CMD > gpurun_out/f/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct --clock-control none -k regex:"pa_quad|pa_fast|classify" -s 12 -c 4 --csv --log-file gpurun_out/f/m.csv $CMD > gpurun_out/f/ncu.log 2>&1
echo ncu rc=$?
