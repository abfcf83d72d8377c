cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/bits
cat > /tmp/bt2.py <<'PY'
import sys, torch
sys.path.insert(0, '.')
import paper_1002_1168_b200 as me
from paper_1002_1168_b200 import batch as B, synth
luma, alpha = synth.config4_batch_dev(256, 20260000, 30)
bits, binary = B.pack_mask_dev(alpha)
cfg = me.BatchConfig(algo=me.Algo.PA, search=me.SearchConfig(search_range=16, block_size=8))
recs = torch.empty((256, 28, 36, 44, 16), dtype=torch.uint8, device='cuda'); stats = torch.empty((256, 28, 48), dtype=torch.uint8, device='cuda')
for _ in range(2):
    B.run_sequences_dev(cfg, luma, alpha, recs, stats)
    B.run_sequences_bits_dev(cfg, luma, bits, recs, stats)
torch.cuda.synchronize()
print("ok")
PY
python /tmp/bt2.py > gpurun_out/bits/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,launch__registers_per_thread --clock-control none -k regex:"classify" --csv --log-file gpurun_out/bits/m.csv python /tmp/bt2.py > gpurun_out/bits/ncu.log 2>&1
echo rc=$?
