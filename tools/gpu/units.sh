cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/units
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29543 bench.py --gpus 2 --dist-backend gloo --same-device --workload cfg3-fss --steps 3 --warmup 3 --es-steps 3 > gpurun_out/units/fss2.json 2>gpurun_out/units/fss2.log; echo rc=$?; tail -2 gpurun_out/units/fss2.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29544 bench.py --gpus 2 --dist-backend gloo --same-device --workload cfg2-es --steps 3 --warmup 3 --es-steps 3 > gpurun_out/units/es2.json 2>gpurun_out/units/es2.log; echo rc=$?; tail -2 gpurun_out/units/es2.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-critical --no-bits > gpurun_out/units/def.json 2>gpurun_out/units/def.log; echo rc=$?; tail -2 gpurun_out/units/def.log
