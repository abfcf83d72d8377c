python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "es or golden or full_search or block_search" > gpurun_out/es_tests.log 2>&1; tail -2 gpurun_out/es_tests.log
python bench.py --workload cfg5-es --no-cpu --steps 3 --warmup 3 > gpurun_out/es_bench.json 2> gpurun_out/es_bench.err
python -c "import json; d=json.load(open('gpurun_out/es_bench.json')); print(d['ms_per_step'], d['roofline']['frac'], d['parity'])"
