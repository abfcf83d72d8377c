set -x
cd $GRAFT_REPO_ROOT
python bench.py --steps 20 --warmup 3 > gpurun_out/b_cfg4.json 2> gpurun_out/b_cfg4.log; echo rc=$?
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/b_ref.json 2> gpurun_out/b_ref.log; echo rc=$?
timeout 300 python bench.py --workload cfg5-es --frames 4 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/b_cfg5es.json 2> gpurun_out/b_cfg5es.log; echo rc=$?
timeout 300 python bench.py --workload cfg2-pa --steps 20 --warmup 3 --no-cpu > gpurun_out/b_cfg2pa.json 2> gpurun_out/b_cfg2pa.log; echo rc=$?
python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu.log 2>&1; echo rc=$?
tail -3 gpurun_out/*.log
