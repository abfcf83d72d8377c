cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q --timeout 300 -x 2>&1 | tail -15
timeout 300 python bench.py --steps 50 --warmup 3 --no-cpu > gpurun_out/q_cfg4.json 2> gpurun_out/q_cfg4.log; echo rc=$?
timeout 300 python bench.py --workload cfg2-pa --steps 50 --warmup 3 --no-cpu --no-e2e > gpurun_out/q_cfg2pa.json 2> gpurun_out/q_cfg2pa.log; echo rc=$?
python - <<'PY'
import json
for f in ["q_cfg4","q_cfg2pa"]:
    try:
        d=json.load(open(f"gpurun_out/{f}.json"))
        print(f, "ms/step %.3f"%d["ms_per_step"], "value %.3g"%d["value"], "stages", {k:round(v,3) for k,v in d["stages_ms"].items()}, "roof", d["roofline"]["frac"], "e2e", d["e2e"] and "%.3g"%d["e2e"]["value"], "clk", d["clocks"])
    except Exception as e: print(f, "ERR", e)
PY
