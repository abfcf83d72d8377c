"""Batched sequence pipeline (the benchmark path): the frame-pair loop of the
reference's run_experiment (proj/src/bench.cpp:155-205) over many sequences at
once, fully on the GPU (me_b200_run_sequences_dev / me_b200_run_sequences).

torch is used only for device memory and streams; the compute is the C ABI.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from ._lib import MeConfig, check, ctx, lib
from .api import Algo, BoundaryTemporal, PrsConfig, SearchConfig, _cfg


@dataclass
class BatchConfig:
    algo: Algo = Algo.PA
    search: SearchConfig = None
    prs: PrsConfig = None
    boundary_temporal: BoundaryTemporal = BoundaryTemporal.Texture

    def __post_init__(self):
        if self.search is None:
            self.search = SearchConfig()
        if self.prs is None:
            self.prs = PrsConfig()

    def c(self) -> MeConfig:
        return _cfg(self.algo, self.search, self.prs, self.boundary_temporal)


def rec_view(t):
    """Views a uint8 torch/numpy buffer of records as the me_block_rec dtype."""
    a = t.cpu().numpy() if hasattr(t, "cpu") else t
    return a.view(_lib.rec_dtype())


def run_sequences_dev(cfg: BatchConfig, luma, alpha=None, recs=None, stats=None, pred=None, device: int = 0, stream=None):
    """Device-resident inputs: luma/alpha are uint8 CUDA tensors [n_seq, F, H, W].

    Returns (recs, stats) as uint8 CUDA tensors of shape [n_seq, pairs, rows,
    cols, 16] and [n_seq, pairs, 48] (views via ``rec_view``); enqueued on
    ``stream`` (torch's current stream when None), not synchronised.
    """
    import torch

    n_seq, F, H, W = luma.shape
    bs = cfg.search.block_size
    pairs = F - cfg.search.ref_distance
    rows, cols = H // bs, W // bs
    if recs is None:
        recs = torch.empty((n_seq, pairs, rows, cols, 16), dtype=torch.uint8, device=luma.device)
    if stats is None:
        stats = torch.empty((n_seq, pairs, 48), dtype=torch.uint8, device=luma.device)
    _check_dev_buffers(luma, alpha, recs, stats, pred, device, (n_seq, pairs, rows, cols, 16), (n_seq, pairs, 48), (n_seq, pairs, H, W))
    if stream is None:
        stream = torch.cuda.current_stream(luma.device).cuda_stream
    c = cfg.c()
    check(
        lib().me_b200_run_sequences_dev(
            ctx(device), C.byref(c), n_seq, F, W, H,
            C.c_void_p(luma.data_ptr()),
            C.c_void_p(alpha.data_ptr()) if alpha is not None else None,
            C.c_void_p(recs.data_ptr()), C.c_void_p(stats.data_ptr()),
            C.c_void_p(pred.data_ptr()) if pred is not None else None,
            C.c_void_p(stream),
        )
    )
    return recs, stats


def _check_dev_buffers(luma, alpha, recs, stats, pred, device, recs_shape, stats_shape, pred_shape):
    """The C ABI takes raw device pointers: wrong dtype, strides, device or
    sizes would be silently misread (or written out of bounds), so check here."""
    import torch

    def chk(name, t, shape):
        if t is None:
            return
        if t.dtype != torch.uint8 or not t.is_contiguous() or t.device.type != "cuda" or t.device.index != device:
            raise ValueError(f"{name}: need a contiguous uint8 tensor on cuda:{device}")
        if tuple(t.shape) != tuple(shape):
            raise ValueError(f"{name}: shape {tuple(t.shape)} != {tuple(shape)}")

    chk("luma", luma, luma.shape)
    chk("alpha", alpha, luma.shape)
    chk("recs", recs, recs_shape)
    chk("stats", stats, stats_shape)
    chk("pred", pred, pred_shape)


def pack_mask_dev(alpha, device: int = 0, stream=None):
    """Device mask bytes [..., H, W] -> (bit plane uint8 [..., H, W // 8] with
    bit i of byte j = pel 8j + i, binary): me_b200_pack_mask_dev.  The bit
    form is exact when `binary` (every byte 0 or 255)."""
    import torch

    if alpha.dtype != torch.uint8 or not alpha.is_contiguous() or alpha.numel() % 64:
        raise ValueError("alpha: contiguous uint8 CUDA tensor with a multiple of 64 elements")
    bits = torch.empty(alpha.shape[:-1] + (alpha.shape[-1] // 8,), dtype=torch.uint8, device=alpha.device)
    if stream is None:
        stream = torch.cuda.current_stream(alpha.device).cuda_stream
    flag = C.c_int()
    check(lib().me_b200_pack_mask_dev(ctx(device), C.c_void_p(alpha.data_ptr()), alpha.numel(), C.c_void_p(bits.data_ptr()), C.byref(flag), C.c_void_p(stream)))
    return bits, bool(flag.value)


def run_sequences_bits_dev(cfg: BatchConfig, luma, alpha_bits, recs=None, stats=None, pred=None, device: int = 0, stream=None):
    """run_sequences_dev with BINARY masks as device bit planes
    (me_b200_run_sequences_bits_dev): alpha_bits [n_seq, F, H, W // 8]."""
    import torch

    n_seq, F, H, W = luma.shape
    bs = cfg.search.block_size
    pairs = F - cfg.search.ref_distance
    rows, cols = H // bs, W // bs
    if recs is None:
        recs = torch.empty((n_seq, pairs, rows, cols, 16), dtype=torch.uint8, device=luma.device)
    if stats is None:
        stats = torch.empty((n_seq, pairs, 48), dtype=torch.uint8, device=luma.device)
    _check_dev_buffers(luma, None, recs, stats, pred, device, (n_seq, pairs, rows, cols, 16), (n_seq, pairs, 48), (n_seq, pairs, H, W))
    if alpha_bits.dtype != torch.uint8 or not alpha_bits.is_contiguous() or tuple(alpha_bits.shape) != (n_seq, F, H, W // 8):
        raise ValueError("alpha_bits: contiguous uint8 [n_seq, F, H, W // 8]")
    if stream is None:
        stream = torch.cuda.current_stream(luma.device).cuda_stream
    c = cfg.c()
    check(lib().me_b200_run_sequences_bits_dev(ctx(device), C.byref(c), n_seq, F, W, H, C.c_void_p(luma.data_ptr()), C.c_void_p(alpha_bits.data_ptr()),
                                               C.c_void_p(recs.data_ptr()), C.c_void_p(stats.data_ptr()),
                                               C.c_void_p(pred.data_ptr()) if pred is not None else None, C.c_void_p(stream)))
    return recs, stats


def run_band_dev(cfg: BatchConfig, luma, alpha, row0: int, row1: int, recs, stats, device: int = 0, stream=None):
    """The block-row band [row0, row1) of a device-resident batch
    (me_b200_run_band_dev; baselines only): writes the band's records, and its
    share of each pair's stats into `stats` (zeroed first by the library)."""
    import torch

    n_seq, F, H, W = luma.shape
    bs = cfg.search.block_size
    pairs = F - cfg.search.ref_distance
    _check_dev_buffers(luma, alpha, recs, stats, None, device, (n_seq, pairs, H // bs, W // bs, 16), (n_seq, pairs, 48), None)
    if stream is None:
        stream = torch.cuda.current_stream(luma.device).cuda_stream
    c = cfg.c()
    check(lib().me_b200_run_band_dev(ctx(device), C.byref(c), n_seq, F, W, H, C.c_void_p(luma.data_ptr()),
                                     C.c_void_p(alpha.data_ptr()) if alpha is not None else None, int(row0), int(row1),
                                     C.c_void_p(recs.data_ptr()), C.c_void_p(stats.data_ptr()), C.c_void_p(stream)))
    return recs, stats


def run_sequences_multi(cfg: BatchConfig, luma: np.ndarray, alpha: Optional[np.ndarray] = None, n_gpus: int = 1):
    """me_b200_run_sequences_multi: the host batch sharded over n_gpus devices
    of this process (sequences, or a single baseline sequence's frame pairs)."""
    luma = np.ascontiguousarray(luma, np.uint8)
    if luma.ndim == 3:
        luma = luma[None]
    n_seq, F, H, W = luma.shape
    if alpha is not None:
        alpha = np.ascontiguousarray(alpha, np.uint8).reshape(luma.shape)
    bs = cfg.search.block_size
    pairs = F - cfg.search.ref_distance
    recs = np.zeros((n_seq, pairs, H // bs, W // bs), _lib.rec_dtype())
    stats = np.zeros((n_seq, pairs), _lib.stats_dtype())
    c = cfg.c()
    vp = lambda a: None if a is None else a.ctypes.data_as(C.c_void_p)
    check(lib().me_b200_run_sequences_multi(C.byref(c), n_seq, F, W, H, vp(luma), vp(alpha), vp(recs), vp(stats), int(n_gpus)))
    return recs, stats


def run_sequences(cfg: BatchConfig, luma: np.ndarray, alpha: Optional[np.ndarray] = None, want_pred: bool = False, device: int = 0):
    """End to end from host arrays [n_seq, F, H, W] (pinned or pageable):
    H2D, device pipeline, D2H.  Returns (recs, stats[, pred]) numpy arrays."""
    luma = np.ascontiguousarray(luma, np.uint8)
    if luma.ndim == 3:
        luma = luma[None]
    n_seq, F, H, W = luma.shape
    if alpha is not None:
        alpha = np.ascontiguousarray(alpha, np.uint8).reshape(luma.shape)
    bs = cfg.search.block_size
    pairs = F - cfg.search.ref_distance
    if pairs < 1:
        raise ValueError("ref_distance must be smaller than the frame count")
    recs = np.zeros((n_seq, pairs, H // bs, W // bs), _lib.rec_dtype())
    stats = np.zeros((n_seq, pairs), _lib.stats_dtype())
    pred = np.zeros((n_seq, pairs, H, W), np.uint8) if want_pred else None
    c = cfg.c()
    vp = lambda a: None if a is None else a.ctypes.data_as(C.c_void_p)
    check(lib().me_b200_run_sequences(ctx(device), C.byref(c), n_seq, F, W, H, vp(luma), vp(alpha), vp(recs), vp(stats), vp(pred)))
    if want_pred:
        return recs, stats, pred
    return recs, stats


def run_sequences_ptr(cfg: BatchConfig, n_seq: int, F: int, W: int, H: int, luma_ptr: int, alpha_ptr: Optional[int], recs_ptr: int, stats_ptr: int, device: int = 0):
    """Raw host-pointer form (e.g. pinned torch tensors) for end-to-end timing."""
    c = cfg.c()
    check(lib().me_b200_run_sequences(ctx(device), C.byref(c), n_seq, F, W, H, C.c_void_p(luma_ptr), C.c_void_p(alpha_ptr) if alpha_ptr else None, C.c_void_p(recs_ptr), C.c_void_p(stats_ptr), None))


def last_transfer_bytes(device: int = 0):
    """(host->device, device->host) bytes of the last run_sequences call on this
    thread's context; binary alpha masks cross PCIe bit-packed."""
    h, d = C.c_int64(), C.c_int64()
    check(lib().me_b200_ctx_transfer_bytes(ctx(device), C.byref(h), C.byref(d)))
    return h.value, d.value


def last_launches(device: int = 0) -> int:
    """Kernels launched by the last batched call on this thread's context."""
    n = C.c_int64()
    check(lib().me_b200_ctx_launches(ctx(device), C.byref(n)))
    return n.value
