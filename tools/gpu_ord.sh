cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_golden.py -m gpu -q --timeout 100 -x 2>&1 | tail -2
ME_PA_MODE=quad ME_PA_QMINB=3 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 100 -x 2>&1 | tail -2
bash tools/gpu_sweep.sh "ME_FILL_ORDER=0" "ME_FILL_ORDER=1" "ME_FILL_ORDER=0 ME_PA_MODE=quad ME_PA_QMINB=3" "ME_PA_MODE=quad ME_PA_QMINB=3" "ME_PA_MODE=quad ME_PA_QMINB=2" "ME_PA_MODE=duo"
