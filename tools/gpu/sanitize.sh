cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/san
TOOL=${1:-racecheck}
timeout 300 python tools/sanitize_run.py > gpurun_out/san/plain.log 2>&1 && \
timeout 1500 compute-sanitizer --tool $TOOL --print-limit 50 python tools/sanitize_run.py > gpurun_out/san/$TOOL.log 2>&1
echo rc=$?
tail -15 gpurun_out/san/$TOOL.log
