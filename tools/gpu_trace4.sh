cd $GRAFT_REPO_ROOT
ME_PA_MODE=${MODE:-duo} ME_PA_TRACE=gpurun_out/trace_cfg4.bin timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e > /dev/null 2>gpurun_out/t4.log; echo rc=$?
ls -la gpurun_out/trace_cfg4.bin
