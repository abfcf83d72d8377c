"""Pins the CPU oracle restatement (oracle/me_oracle.c) to the UNMODIFIED
reference (oracle/_ref/libme_ref.so, compiled from /root/reference/proj/src)
on fresh seeded inputs beyond the stored goldens: every algorithm, both block
sizes, half-pel mode, shape-scored temporal candidates, PRS parameter
variants.  Skipped where oracle/_ref is not built (the GPU box)."""
import numpy as np
import pytest

import oracle
from paper_1002_1168_b200 import synth


@pytest.mark.parametrize("cid,seed,frames", [(1, 21, None), (2, 22, 7)])
@pytest.mark.parametrize("algo,bs,extra", [
    (4, 8, {}), (4, 16, {}), (4, 8, {"halfpel": 1}), (4, 8, {"boundary_temporal": 1}),
    (4, 8, {"max_iterations": 2}), (4, 16, {"max_iterations": 6, "epsilon": 0.25, "theta": 1.0}),
    (0, 16, {}), (1, 16, {}), (2, 16, {}), (3, 16, {}), (3, 8, {"search_range": 5}),
])
def test_sequences_port_equals_reference(port, refo, cid, seed, frames, algo, bs, extra):
    luma, alpha = synth.config_sequence(cid, seed, frames)
    kw = dict(algo=algo, search_range=16, block_size=bs)
    kw.update(extra)
    cfg = oracle.make_cfg(**kw)
    r1, s1 = refo.run_sequence(cfg, luma, alpha)
    r2, s2 = port.run_sequence(cfg, luma, alpha)
    assert np.array_equal(r1, r2) and np.array_equal(s1, s2)


def test_no_mask_and_prediction(port, refo):
    luma, _ = synth.config_sequence(1, 31, 5)
    for algo, bs in ((4, 8), (0, 16), (3, 16)):
        cfg = oracle.make_cfg(algo=algo, search_range=7, block_size=bs, ref_distance=1)
        r1, s1, p1 = refo.run_sequence(cfg, luma, None, want_pred=True)
        r2, s2, p2 = port.run_sequence(cfg, luma, None, want_pred=True)
        assert np.array_equal(r1, r2) and np.array_equal(s1, s2) and np.array_equal(p1, p2)


def test_errors_match(port, refo):
    f = np.zeros((32, 32), np.uint8)
    for o in (port, refo):
        with pytest.raises(oracle.OracleError) as e:
            o.block_search(0, f, f, 24, 24, 16, 7)  # rect outside the frame
        assert e.value.code == 1
        with pytest.raises(oracle.OracleError) as e:
            o.sad_shape(f, f, 0, 0, 16, 1, 0)  # half-pel shape SAD
        assert e.value.code == 1
        with pytest.raises(oracle.OracleError) as e:
            o.brs_select(f, f, None, None, 0, 0, 16, 2, [0] * 8, 7)  # boundary without masks
        assert e.value.code == 1
