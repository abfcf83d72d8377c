cd $GRAFT_REPO_ROOT
CMD="python bench.py --workload cfg2-pa --steps 3 --warmup 3 --no-e2e --no-cpu"
export ME_PA_KEY_A=1 ME_PA_KEY_S=0
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pa_lane_kernel" -s 3 -c 1 -o gpurun_out/prof_pa2 $CMD > gpurun_out/prof_ncu.log 2>&1
echo rc=$?
