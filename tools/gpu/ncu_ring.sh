cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ring4
for w in cfg5-tss cfg3-fss; do
CMD="python bench.py --workload $w --steps 2 --warmup 3 --no-e2e --no-cpu --no-parity --no-es"
$CMD > gpurun_out/ring4/plain_$w.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"ring_kernel" -s 3 -c 1 -o gpurun_out/ring4/prof_$w $CMD > gpurun_out/ring4/ncu_$w.log 2>&1; echo $w rc=$?
done
