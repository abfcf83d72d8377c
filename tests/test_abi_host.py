"""CPU-side checks of the product: the C-ABI library loads and exports every
symbol include/me_b200.h declares, refuses compute without an sm_100 device
(no CPU fallback), validates like the reference, and the host-side mirror
logic (window clipping, candidate gathering, PSNR tail, names) matches the
reference semantics."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

import paper_1002_1168_b200 as me
from paper_1002_1168_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    text = open(os.path.join(ROOT, "include", "me_b200.h")).read()
    return sorted(set(re.findall(r"\b(me_b200_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = C.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 24
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)


def test_version_and_config_validation():
    L = me.lib()
    assert b"sm_100a" in L.me_b200_version()
    good = _lib.MeConfig(4, 16, 8, 2, 0, 4, 2, 0, 0.5, 2.0)
    assert L.me_b200_validate_config(C.byref(good)) == 0
    bad_cases = [
        (dict(search_range=0), "search_range"),
        (dict(block_size=12), "block_size"),
        (dict(ref_distance=0), "ref_distance"),
        (dict(epsilon=0.0), "epsilon"),
        (dict(theta=0.0), "theta"),
        (dict(max_iterations=0), "max_iterations"),
        (dict(step=3), "step"),
        (dict(algo=7), "algorithm"),
    ]
    for kw, word in bad_cases:
        c = _lib.MeConfig(4, 16, 8, 2, 0, 4, 2, 0, 0.5, 2.0)
        for k, v in kw.items():
            setattr(c, k, v)
        assert L.me_b200_validate_config(C.byref(c)) == _lib.ME_ERR_INVALID_ARGUMENT
        assert word in L.me_b200_last_error().decode()


@pytest.mark.skipif(me.device_count() > 0, reason="checks the no-device behaviour")
def test_no_cpu_fallback():
    L = me.lib()
    h = C.c_void_p()
    assert L.me_b200_ctx_create(0, C.byref(h)) == _lib.ME_ERR_NO_DEVICE
    with pytest.raises(RuntimeError):
        me.full_search(np.zeros((32, 32), np.uint8), np.zeros((32, 32), np.uint8), me.BlockRect(0, 0, 16), me.SearchConfig(block_size=16), me.SearchStats())


def test_host_mirror_semantics():
    # clip_to_window (test_estimators.cpp:77-97)
    inner, corner, last = me.BlockRect(24, 24, 16), me.BlockRect(0, 0, 16), me.BlockRect(48, 48, 16, 3, 3)
    assert me.clip_to_window((6, -4), inner, 64, 64, 7) == (6, -4)
    assert me.clip_to_window((-10, -10), corner, 64, 64, 7) == (0, 0)
    assert me.clip_to_window((20, 0), corner, 64, 64, 7) == (14, 0)
    assert me.clip_to_window((10, 10), last, 64, 64, 7) == (0, 0)
    assert me.clip_to_window((3, -1), inner, 64, 64, 7) == (3, -1)
    # gather_candidates (test_estimators.cpp:191-237)
    f = me.MotionField(4, 3, 16)
    prev = me.MotionField(4, 3, 16)
    f.set(0, 1, (2, 0)); f.set(1, 0, (4, 0)); f.set(2, 0, (6, 0)); prev.set(1, 1, (8, 0))
    cs = me.gather_candidates(f, prev, 1, 1)
    assert (cs.a, cs.b, cs.c, cs.t) == ((2, 0), (4, 0), (6, 0), (8, 0))
    assert me.gather_candidates(f, None, 0, 0) == me.CandidateSet()
    f.set(3, 0, (10, 0)); f.set(2, 1, (12, 0))
    cs = me.gather_candidates(f, prev, 3, 1)
    assert cs.a == (12, 0) and cs.b == (10, 0) and cs.c == (0, 0)
    with pytest.raises(ValueError):
        me.gather_candidates(f, me.MotionField(2, 2, 16), 1, 1)
    with pytest.raises(IndexError):
        me.gather_candidates(f, None, 4, 0)
    # names, configs, grid
    assert [me.algo_from_string(me.to_string(a)) for a in me.Algo] == list(me.Algo)
    assert me.algo_from_string("4ss") == me.Algo.FSS
    with pytest.raises(ValueError):
        me.algo_from_string("NSTSS")
    with pytest.raises(ValueError):
        me.SearchConfig(block_size=12).validate()
    with pytest.raises(ValueError):
        me.PrsConfig(step=3).validate()
    assert len(me.block_grid(176, 144, 16)) == 99
    with pytest.raises(ValueError):
        me.block_grid(100, 100, 16)
    with pytest.raises(ValueError):
        me.MotionField(0, 3)


def test_psnr_tail_and_figure_of_merit():
    # metrics.cpp:117-123 on a GPU-computed SSE: mse = 1 -> 48.1308 dB
    r = me.psnr_from_sse(32 * 32, 32 * 32)
    assert r.mse == 1.0 and abs(r.psnr_db - 48.1308) < 1e-4 and r.psnr_linear == 65025.0
    assert me.psnr_from_sse(0, 100).infinite()
    assert r.psnr_db == 10.0 * math.log10(255.0 * 255.0 / 1.0)
    assert me.figure_of_merit(1000.0, 7, 5.0) == 1000.0 * 225 / 5.0
    with pytest.raises(ValueError):
        me.figure_of_merit(1.0, 0, 1.0)
    # residual helpers (host, off the hot path)
    a, b = np.full((4, 4), 10, np.uint8), np.full((4, 4), 250, np.uint8)
    assert (me.residual(a, b) == -240).all()
    assert (me.residual_to_gray(me.residual(a, b)) == 0).all()


def _decode_sparse_mask(buf: np.ndarray, n: int) -> np.ndarray:
    """numpy restatement of the transfer form documented at me_b200_pack_mask."""
    nwords = n // 64
    groups = (nwords + 31) // 32
    pres = buf[: 4 * groups].view(np.uint32)
    base = buf[4 * groups: 8 * groups].view(np.uint32)
    head = (8 * groups + 15) & ~15
    words = np.zeros(nwords, np.uint64)
    lit = buf[head:].view(np.uint64)
    for g in range(groups):
        m = int(pres[g])
        k = int(base[g])
        for i in range(32):
            if (m >> i) & 1:
                words[32 * g + i] = lit[k]
                k += 1
    bits = np.unpackbits(words.view(np.uint8), bitorder="little")
    return (bits * 255).astype(np.uint8)


@pytest.mark.parametrize("n", [64, 2048, 4096 + 64, 352 * 288 * 3])
def test_pack_mask_roundtrip(n):
    """The host path's sparse bit-packed mask (zero 64-pixel words elided)
    decodes back to the mask; non-binary masks and bad sizes are refused."""
    L = me.lib()
    rng = np.random.default_rng(n)
    mask = np.zeros(n, np.uint8)
    for _ in range(max(1, n // 5000)):  # a few runs of foreground, like object masks
        a = int(rng.integers(0, n))
        mask[a: a + int(rng.integers(1, 700))] = 255
    mask[rng.integers(0, n, size=max(1, n // 1000))] = 255  # and isolated pixels
    cap = 16 + n // 256 + n // 8 + 64
    out = np.zeros(cap, np.uint8)
    nb = C.c_size_t(0)
    assert L.me_b200_pack_mask(mask.ctypes.data, n, out.ctypes.data, cap, C.byref(nb)) == 0
    assert nb.value <= cap
    assert np.array_equal(_decode_sparse_mask(out[: nb.value], n), mask)
    gray = mask.copy()
    gray[n // 2] = 7
    assert L.me_b200_pack_mask(gray.ctypes.data, n, out.ctypes.data, cap, C.byref(nb)) == _lib.ME_ERR_INVALID_ARGUMENT
    assert "binary" in L.me_b200_last_error().decode()
    assert L.me_b200_pack_mask(mask.ctypes.data, n - 8, out.ctypes.data, cap, C.byref(nb)) == _lib.ME_ERR_INVALID_ARGUMENT


def test_ctypes_structs_match_the_header(tmp_path):
    """The ctypes mirrors of the C ABI structs (_lib) have the header's size and
    field offsets (gcc on include/me_b200.h)."""
    import ctypes as C
    import subprocess

    from paper_1002_1168_b200 import _lib

    structs = {"me_tuning": _lib.MeTuning, "me_config": _lib.MeConfig}
    src = ['#include <stddef.h>', '#include <stdio.h>', '#include "me_b200.h"', "int main(void) {"]
    for cname, py in structs.items():
        src.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f, _ in py._fields_:
            src.append(f'printf("{cname} {f} %zu\\n", offsetof({cname}, {f}));')
    src.append("return 0; }")
    (tmp_path / "l.c").write_text("\n".join(src))
    inc = os.path.join(ROOT, "include")
    subprocess.run(["gcc", "-I", inc, str(tmp_path / "l.c"), "-o", str(tmp_path / "l")], check=True)
    got = subprocess.run([str(tmp_path / "l")], capture_output=True, text=True, check=True).stdout.split("\n")
    for line in filter(None, got):
        cname, field, val = line.split()
        py = structs[cname]
        want = C.sizeof(py) if field == "size" else getattr(py, field).offset
        assert int(val) == want, f"{cname}.{field}: C {val} vs ctypes {want}"
