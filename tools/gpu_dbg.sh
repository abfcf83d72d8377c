cd $GRAFT_REPO_ROOT
ME_PA_DBG=1 ME_PA_KEY_A=1 ME_PA_KEY_S=0 timeout 120 python bench.py --workload cfg2-pa --steps 1 --warmup 3 --no-cpu --no-e2e 2>&1 >/dev/null | grep "pa dbg" | tail -1
ME_PA_DBG=1 ME_PA_KEY_A=1 ME_PA_KEY_S=0 timeout 120 python bench.py --workload cfg4-pa --steps 1 --warmup 3 --no-cpu --no-e2e 2>&1 >/dev/null | grep "pa dbg" | tail -1
