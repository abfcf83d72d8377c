# Evidence refresh without the (unchanged-kernel) ncu --set full captures.
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ev
python bench.py > gpurun_out/ev/bench_default.json 2> gpurun_out/ev/bench_default.log; echo bench rc=$?
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ev/bench_ref.json 2> gpurun_out/ev/bench_ref.log; echo ref rc=$?
timeout 300 python bench.py --workload cfg2-pa --steps 50 --warmup 5 > gpurun_out/ev/bench_cfg2pa.json 2> gpurun_out/ev/bench_cfg2pa.log; echo cfg2 rc=$?
timeout 300 python bench.py --workload cfg5-es --frames 4 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/ev/bench_cfg5es.json 2> gpurun_out/ev/bench_cfg5es.log; echo cfg5 rc=$?
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/ev/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/ev/launches.csv $CMD > gpurun_out/ev/ncu_launch.log 2>&1; echo launches rc=$?
python -c "import json;d=json.load(open('gpurun_out/ev/bench_default.json'));print(d['ms_per_step'], d['value'], d['stages_ms'], d['e2e'], d['clocks'])"
