# The multi-rank bench path (strong-sharded config 4 + per-step gather of MVs/stats,
# rank-0 parity of the whole batch, ES (pair, row-band) units) with 2 ranks on ONE GPU:
# gloo collectives through the host; the timings are meaningless (shared GPU).
cd $GRAFT_REPO_ROOT
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 \
  bench.py --gpus 2 --dist-backend gloo --same-device --steps 3 --warmup 3 --e2e-steps 2 --es-steps 2 > /tmp/two.json 2> /tmp/two.log
echo rc=$?
tail -5 /tmp/two.log
python -c "
import json; d=json.load(open('/tmp/two.json'))
print(d['n_gpus'], d['scaling'], d['config']['sequences'], d['parity'], d['es_cfg5']['parity'], d['es_cfg5']['units'], d['bits_layout']['identical_to_byte_masks'])"
