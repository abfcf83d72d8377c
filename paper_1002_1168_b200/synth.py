"""Seeded synthetic inputs for BASELINE.json configs 1..5, from the
deterministic integer generator in csrc/synth.cpp (me_b200_synth)."""
from __future__ import annotations

import ctypes as C
from concurrent.futures import ThreadPoolExecutor
from typing import Optional, Tuple

import numpy as np

from ._lib import MeSynthParams, check, lib

# (search_range, algorithms) per config, BASELINE.json "configs"
CONFIG_SEARCH = {1: 16, 2: 16, 3: 32, 4: 16, 5: 64}


def preset(config_id: int, seed: int, frames: Optional[int] = None, size: Optional[Tuple[int, int]] = None) -> MeSynthParams:
    p = MeSynthParams()
    check(lib().me_b200_synth_preset(int(config_id), C.c_uint64(seed), C.byref(p)))
    if frames is not None:
        p.frames = int(frames)
    if size is not None:
        p.width, p.height = int(size[0]), int(size[1])
    return p


def generate(p: MeSynthParams, out_luma: Optional[np.ndarray] = None, out_alpha: Optional[np.ndarray] = None):
    """Returns (luma, alpha) uint8 arrays [frames, H, W]."""
    shape = (p.frames, p.height, p.width)
    luma = np.empty(shape, np.uint8) if out_luma is None else out_luma
    alpha = np.empty(shape, np.uint8) if out_alpha is None else out_alpha
    assert luma.shape == shape and alpha.shape == shape and luma.flags.c_contiguous and alpha.flags.c_contiguous
    check(lib().me_b200_synth(C.byref(p), luma.ctypes.data_as(C.c_void_p), alpha.ctypes.data_as(C.c_void_p)))
    return luma, alpha


def config_sequence(config_id: int, seed: int, frames: Optional[int] = None, size=None):
    return generate(preset(config_id, seed, frames, size))


def config4_batch(n_seq: int, base_seed: int, frames: Optional[int] = None, luma: Optional[np.ndarray] = None, alpha: Optional[np.ndarray] = None, threads: int = 8):
    """n_seq config-2 sequences with seed = base + i (config 4), generated in
    parallel (the C generator releases the GIL)."""
    p0 = preset(4, base_seed, frames)
    shape = (n_seq, p0.frames, p0.height, p0.width)
    if luma is None:
        luma = np.empty(shape, np.uint8)
    if alpha is None:
        alpha = np.empty(shape, np.uint8)

    def one(i):
        generate(preset(4, base_seed + i, frames), luma[i], alpha[i])

    with ThreadPoolExecutor(max(1, threads)) as ex:
        list(ex.map(one, range(n_seq)))
    return luma, alpha


def config4_batch_dev(n_seq: int, base_seed: int, frames: Optional[int] = None, config_id: int = 4, device: int = 0, stream=None):
    """The same batch generated on the GPU (me_b200_synth_dev): uint8 CUDA
    tensors (luma, alpha) [n_seq, frames, H, W], byte-identical to
    config4_batch."""
    import torch

    from ._lib import ctx

    params = (MeSynthParams * n_seq)()
    for i in range(n_seq):
        params[i] = preset(config_id, base_seed + i, frames)
    p0 = params[0]
    shape = (n_seq, p0.frames, p0.height, p0.width)
    dev = torch.device("cuda", device)
    luma = torch.empty(shape, dtype=torch.uint8, device=dev)
    alpha = torch.empty(shape, dtype=torch.uint8, device=dev)
    if stream is None:
        stream = torch.cuda.current_stream(dev).cuda_stream
    check(lib().me_b200_synth_dev(ctx(device), params, n_seq, C.c_void_p(luma.data_ptr()), C.c_void_p(alpha.data_ptr()), C.c_void_p(stream)))
    return luma, alpha
