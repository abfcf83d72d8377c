# ES changes: the ES/baseline GPU tests, then the config-2 and config-5 ES lines
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/es
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "es or golden or full_search or block_search or sequence or band or fuzz or range" > gpurun_out/es/tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/es/tests.log
timeout 600 python bench.py --workload cfg2-es --steps 200 --warmup 5 --no-es > gpurun_out/es/cfg2.json 2> gpurun_out/es/cfg2.log; echo cfg2 rc=$?
timeout 600 python bench.py --workload cfg5-es --steps 3 --warmup 3 --no-es > gpurun_out/es/cfg5.json 2> gpurun_out/es/cfg5.log; echo cfg5 rc=$?
python - <<'PY'
import json
for w in ("cfg2", "cfg5"):
    try:
        d = json.load(open(f"gpurun_out/es/{w}.json"))
        print(w, round(d["ms_per_step"], 4), d.get("stages_ms"), round(d["roofline"]["frac"], 3), d["parity"])
    except Exception as e:
        print(w, "ERR", e)
PY
