cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/b3
timeout 900 python bench.py > gpurun_out/b3/bench.json 2> gpurun_out/b3/bench.log; echo bench rc=$?
python -c "import json;d=json.load(open('gpurun_out/b3/bench.json'));print(d['ms_per_step'], json.dumps(d['critical_path'])[:1500])"
timeout 600 python bench.py --workload cfg5-es --es-bands 4 --es-steps 3 > gpurun_out/b3/es4.json 2> gpurun_out/b3/es4.log; echo es4 rc=$?
python -c "import json;d=json.load(open('gpurun_out/b3/es4.json'));print(d['ms_per_step'], d['parity'], d['roofline']['frac'])"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 --no-e2e --no-cpu --no-critical > gpurun_out/b3/trun.json 2> gpurun_out/b3/trun.log; echo torchrun rc=$?
python -c "import json;d=json.load(open('gpurun_out/b3/trun.json'));print(d['ms_per_step'], d['n_gpus'], d['scaling'], d['parity'])"
tail -3 gpurun_out/b3/trun.log
