# Round-2 evidence: GPU tests, default bench, reference arm, launch list,
# ncu --set full of the top kernels (each ncu only after the same command ran clean).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ev7
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/ev7/pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/ev7/pytest.log
timeout 900 python bench.py > gpurun_out/ev7/bench.json 2> gpurun_out/ev7/bench.log; echo bench rc=$?
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ev7/ref.json 2> gpurun_out/ev7/ref.log; echo ref rc=$?
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu --no-es --no-parity --no-bits"
$CMD > gpurun_out/ev7/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/ev7/launches.csv $CMD > gpurun_out/ev7/ncu_launch.log 2>&1; echo launches rc=$?
$CMD > gpurun_out/ev7/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pa_quad|classify|pa_fast" -s 12 -c 4 -o gpurun_out/ev7/prof_pa $CMD > gpurun_out/ev7/ncu_pa.log 2>&1; echo ncu_pa rc=$?
CMD2="python bench.py --workload cfg5-es --es-steps 1 --warmup 1 --no-parity --no-cpu"
$CMD2 > gpurun_out/ev7/plain3.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"es_run_kernel|es_kernel" -s 3 -c 1 -o gpurun_out/ev7/prof_es $CMD2 > gpurun_out/ev7/ncu_es.log 2>&1; echo ncu_es rc=$?
