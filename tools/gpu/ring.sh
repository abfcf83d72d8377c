cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/ring5
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 -k "ring or golden or fuzz or band" > gpurun_out/ring5/pytest.log 2>&1; echo pytest rc=$?; tail -2 gpurun_out/ring5/pytest.log
for spec in "cfg3-tss 150" "cfg3-fss 150" "cfg3-ds 150" "cfg5-tss 30" "cfg5-fss 30" "cfg5-ds 30"; do
  set -- $spec
  timeout 900 python bench.py --workload $1 --steps $2 --warmup 5 --no-es --no-e2e --no-cpu > gpurun_out/ring5/$1.json 2> gpurun_out/ring5/$1.log; echo $1 rc=$?
done
