cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/s3base
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 300 > gpurun_out/s3base/pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/s3base/pytest.log
timeout 900 python bench.py > gpurun_out/s3base/bench.json 2> gpurun_out/s3base/bench.log; echo bench rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3base/smoke.log 2>&1; echo smoke rc=$?
