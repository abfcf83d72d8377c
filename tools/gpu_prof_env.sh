# ncu --set full of the PA search kernel under an env setting: gpu_prof_env.sh NAME "ENV..."
cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
env $2 $CMD > gpurun_out/prof_$1.log 2>&1 && \
env $2 ncu --set full --clock-control none --import-source on -k regex:"pa_" -s 3 -c 1 -o gpurun_out/prof_$1 $CMD > gpurun_out/prof_$1_ncu.log 2>&1
echo rc=$?
