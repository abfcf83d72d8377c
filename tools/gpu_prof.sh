cd $GRAFT_REPO_ROOT
export ME_PA_KEY_A=1 ME_PA_KEY_S=0
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/prof_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pa_fast_kernel" -s 3 -c 1 -o gpurun_out/prof_pa $CMD > gpurun_out/prof_ncu.log 2>&1
echo rc=$?
tail -5 gpurun_out/prof_ncu.log
