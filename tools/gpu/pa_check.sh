# A PA kernel change on the GPU: config-4 shards (stage times), the default bench line
# (whole-batch parity vs the reference, critical-path leg) and the PA/sequence GPU tests
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/pc
timeout 600 python tools/key_probe.py 256,128,32 default > gpurun_out/pc/probe.txt 2>&1; echo probe rc=$?
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-es --no-bits > gpurun_out/pc/bench.json 2> gpurun_out/pc/bench.log; echo bench rc=$?
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -k "pa or sequence or golden or batch or fuzz" > gpurun_out/pc/pytest.log 2>&1; echo pytest rc=$?; tail -1 gpurun_out/pc/pytest.log
cat gpurun_out/pc/probe.txt
python - <<'PY'
import json; d = json.load(open("gpurun_out/pc/bench.json"))
print("bench", round(d["ms_per_step"], 4), d["stages_ms"], d["parity"]["mismatches"], {k: round(v["us_per_step"], 3) for k, v in d["critical_path"].items() if isinstance(v, dict)})
PY
