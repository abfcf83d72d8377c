# Every BASELINE config's workload as its own clock-stamped bench line (profiles/r02_lines/)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/lines
for spec in "cfg1-pa 300" "cfg2-pa 200" "cfg2-es 200" "cfg3-pa 30" "cfg3-tss 150" "cfg3-fss 150" "cfg3-ds 150" "cfg5-pa 20" "cfg5-tss 30" "cfg5-fss 30" "cfg5-ds 30"; do
  set -- $spec
  timeout 900 python bench.py --workload $1 --steps $2 --warmup 5 --no-es > gpurun_out/lines/$1.json 2> gpurun_out/lines/$1.log; echo $1 rc=$?
done
