# ncu capture of the ring kernel on the config 5 TSS workload (+ parity of the ring tests first).
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ring_prof
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 200 -x -k "ring or block_search" 2>&1 | tail -2
CMD="python bench.py --workload ${WL:-cfg5-tss} --steps 2 --warmup 3 --no-cpu --no-e2e"
$CMD > gpurun_out/ring_prof/plain.json 2>&1; echo plain rc=$?
ncu --set full --clock-control none --import-source on -k regex:"ring_kernel" -s 2 -c 1 -o gpurun_out/ring_prof/ring_${WL:-cfg5-tss} $CMD > gpurun_out/ring_prof/ncu.log 2>&1; echo ncu rc=$?
tail -3 gpurun_out/ring_prof/ncu.log
