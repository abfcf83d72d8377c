cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/b2
timeout 900 python bench.py > gpurun_out/b2/bench.json 2> gpurun_out/b2/bench.log; echo bench rc=$?
tail -5 gpurun_out/b2/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/b2/ref.json 2> gpurun_out/b2/ref.log; echo ref rc=$?
grep -l libme gpurun_out/b2/ref.log; true
