cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s2
rm -f gpurun_out/s2/prof*.bin
for n in 64 256; do
ME_PA_SEQ_PROF=gpurun_out/s2/prof$n.bin timeout 300 python bench.py --steps 2 --warmup 3 --n-seq $n --no-e2e --no-cpu > /dev/null 2> gpurun_out/s2/b$n.log; echo rc=$?
done
ME_PA_SEQ=1 CUDA_LAUNCH_BLOCKING=1 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k 4gib 2>&1 | tail -5
