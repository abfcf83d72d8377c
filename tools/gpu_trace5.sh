cd $GRAFT_REPO_ROOT
ME_PA_MODE=fast ME_PA_TRACE=gpurun_out/trace_cfg5.bin timeout 300 python bench.py --workload cfg5-pa --frames 6 --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>gpurun_out/t5.log; echo rc=$?
ME_PA_MODE=fast ME_PA_TRACE=gpurun_out/trace_cfg2.bin timeout 300 python bench.py --workload cfg2-pa --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>gpurun_out/t2.log; echo rc=$?
