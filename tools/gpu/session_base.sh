cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s2base
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/s2base/pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/s2base/pytest.log
timeout 900 python bench.py > gpurun_out/s2base/bench.json 2> gpurun_out/s2base/bench.log; echo bench rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2base/smoke.log 2>&1; echo smoke rc=$?
