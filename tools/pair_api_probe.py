"""Per-pair API latency (me_b200_estimate_field, the drop-in's estimate_field):
mean wall time per call for PA (8x8, the previous field as temporal candidates)
and ES (16x16) over a sequence without masks — the quantity the reference's
acceptance criterion 11 compares (recursive faster than exhaustive).
usage: pair_api_probe.py config_id frames [name:field=v,... ...]"""
import sys
import time

sys.path.insert(0, ".")
from paper_1002_1168_b200 import _lib, api, synth  # noqa: E402

cid = int(sys.argv[1]) if len(sys.argv) > 1 else 1
frames = int(sys.argv[2]) if len(sys.argv) > 2 else 50
variants = []
for spec in sys.argv[3:] or ["default"]:
    name, _, kv = spec.partition(":")
    variants.append((name, {k: int(v) for k, v in (x.split("=") for x in kv.split(",") if x)}))
luma, _ = synth.config_sequence(cid, 7, frames)


def run(algo, bs):
    cfg = api.SearchConfig(search_range=16, block_size=bs)
    prs = api.PrsConfig()
    prev, out = None, []
    t0 = time.perf_counter()
    for f in range(2, frames):
        field, st = api.estimate_field(algo, luma[f], luma[f - 2], None, None, prev if algo == api.Algo.PA else None, cfg, prs)
        prev = field
        out.append(field.vectors.copy())
    return (time.perf_counter() - t0) / (frames - 2) * 1e6, out


run(api.Algo.ES, 16)
es_us, _ = run(api.Algo.ES, 16)
print(f"cfg{cid} ES bs16: {es_us:.1f} us per pair", flush=True)
ref = None
for name, kw in variants:
    _lib.set_tuning(0, **kw)
    run(api.Algo.PA, 8)
    us, out = run(api.Algo.PA, 8)
    same = ref is None or all((a == b).all() for a, b in zip(out, ref))
    ref = ref or out
    print(f"cfg{cid} PA bs8 {name}: {us:.1f} us per pair{'' if same else ' DIFFERENT'}", flush=True)
_lib.set_tuning(0)

# the per-pair pipeline's stage times (context events): the search stage of
# a PA pair is the one-CTA shared-memory kernel
import ctypes as C  # noqa: E402

lib, h = _lib.lib(), _lib.ctx(0)
_lib.check(lib.me_b200_ctx_set_profiling(h, 1))
for algo, bs in ((api.Algo.ES, 16), (api.Algo.PA, 8)):
    cfg = api.SearchConfig(search_range=16, block_size=bs)
    acc, n = [0.0] * 4, 0
    prev = None
    for f in range(2, frames):
        field, st = api.estimate_field(algo, luma[f], luma[f - 2], None, None, prev if algo == api.Algo.PA else None, cfg, api.PrsConfig())
        prev = field
        out = (C.c_float * 4)()
        _lib.check(lib.me_b200_ctx_stage_ms(h, out, 4))
        if f > 3:
            acc = [a + x for a, x in zip(acc, out)]
            n += 1
    print(f"cfg{cid} {api.to_string(algo)} stages (classify, sort, search, mc) us:", [round(1000 * a / n, 1) for a in acc], flush=True)
_lib.check(lib.me_b200_ctx_set_profiling(h, 0))
