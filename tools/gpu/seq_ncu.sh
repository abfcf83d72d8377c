cd $GRAFT_REPO_ROOT
CMD="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu"
$CMD > gpurun_out/seqncu_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"pa_seq" -s 2 -c 1 -o gpurun_out/prof_seq $CMD > gpurun_out/prof_seq_ncu.log 2>&1
echo rc=$?
