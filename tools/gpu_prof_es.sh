cd $GRAFT_REPO_ROOT
CMD="python bench.py --workload cfg5-es --frames 4 --steps 1 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/prof_es.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"es_kernel" -s 1 -c 1 -o gpurun_out/prof_es $CMD > gpurun_out/prof_es_ncu.log 2>&1
echo rc=$?
