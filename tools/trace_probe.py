"""Per-block PA trace of a config-4 batch of N sequences (default 32, the
per-GPU shard at 8 GPUs) under the default schedule: runs it once with
me_tuning.pa_trace_path set and prints tools/trace_report.py's analysis."""
import os
import subprocess
import sys

import torch

sys.path.insert(0, ".")
import paper_1002_1168_b200 as me  # noqa: E402
from paper_1002_1168_b200 import _lib, batch as B, synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
sched = sys.argv[2] if len(sys.argv) > 2 else "auto"
extra = dict(kv.split("=") for kv in sys.argv[3:])
extra = {k: int(v) for k, v in extra.items()}
path = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out", f"trace_{n}_{sched}.bin")
cfg = me.BatchConfig(algo=me.Algo.PA, search=me.SearchConfig(search_range=16, block_size=8))
luma, alpha = synth.config4_batch_dev(n, 20260000, 30)
for _ in range(3):
    B.run_sequences_dev(cfg, luma, alpha)
torch.cuda.synchronize()
_lib.set_tuning(0, pa_schedule=sched, pa_trace_path=path, **extra)
B.run_sequences_dev(cfg, luma, alpha)
torch.cuda.synchronize()
_lib.set_tuning(0)
print(n, "sequences,", sched, "schedule,", extra, ":", os.path.getsize(path) if os.path.exists(path) else "no trace file", "bytes")
r = subprocess.run([sys.executable, "tools/trace_report.py", path, "44", "36", "28", "steps"], capture_output=True, text=True)
print(r.stdout, r.stderr)
