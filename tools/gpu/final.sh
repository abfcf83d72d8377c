cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/final
timeout 900 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.log; echo bench rc=$?
timeout 600 python bench.py --impl reference > gpurun_out/final/ref.json 2> gpurun_out/final/ref.log; echo ref rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo smoke rc=$?
