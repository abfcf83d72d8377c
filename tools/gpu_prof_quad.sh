cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
for mb in 3 2; do
export ME_PA_MODE=quad ME_PA_QMINB=$mb
$CMD > gpurun_out/pq$mb.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pa_quad" -s 2 -c 1 -o gpurun_out/prof_quad$mb $CMD > gpurun_out/prof_quad${mb}_ncu.log 2>&1
echo rc=$?
done
