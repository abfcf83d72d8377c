# ncu --set full of pa_quad_kernel with source-level memory counters (cfg4 default bench).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/quad
CMD="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/quad/plain.log 2>&1; echo plain rc=$?
ncu --set full --clock-control none --import-source on -k regex:"pa_quad_kernel" -s 2 -c 1 -o gpurun_out/quad/quad $CMD > gpurun_out/quad/ncu.log 2>&1; echo ncu rc=$?
ncu -i gpurun_out/quad/quad.ncu-rep --page source --csv --print-source sass > gpurun_out/quad/source.csv 2>&1; echo src rc=$?
