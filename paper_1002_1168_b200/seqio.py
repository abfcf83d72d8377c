"""Sequence and mask I/O of the reference (video_io.cpp), host side.

Frames are read whole into pinned-friendly contiguous numpy arrays
(``[frames, H, W]`` luma, chroma optional) so a sequence goes to the GPU in
one batched call.  Formats and error behaviour follow the reference:

* I420 raw (``open_i420``, video_io.cpp:126-138): frame count from the file
  size, which must be a multiple of W*H*3/2.
* Y4M (``open_y4m`` / ``parse_y4m_header``, :79-159): only ``C420*``
  colourspaces, W and H tags required, a fixed-length ``FRAME`` marker.
* P5 PGM masks (``read_pgm``, :194-214; '#' comments skipped) binarised at a
  threshold (``read_mask``, :184-192; ``binarize`` frame.cpp:50-56), file
  names from a printf-style pattern (``MaskSource::path_for``, :71-77).
"""
from __future__ import annotations

import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .api import check_dimensions  # frame.cpp:34-40

I420, Y4M = 0, 1


@dataclass
class SequenceSource:  # video_io.hpp:32-45
    path: str = ""
    format: int = I420
    width: int = 0
    height: int = 0
    frame_count: int = 0
    header_bytes: int = 0
    frame_marker_bytes: int = 0

    def frame_bytes(self) -> int:
        return self.width * self.height * 3 // 2


@dataclass
class MaskSource:  # video_io.hpp:49-55
    pattern: str = ""
    threshold: int = 128

    def present(self) -> bool:
        return bool(self.pattern)

    def path_for(self, index: int) -> str:
        return self.pattern % index


def parse_y4m_header(line: str) -> SequenceSource:
    tags = line.split()
    if not tags or tags[0] != "YUV4MPEG2":
        raise RuntimeError("not a Y4M stream (missing YUV4MPEG2 signature)")
    src = SequenceSource(format=Y4M)
    have_w = have_h = False
    for tag in tags[1:]:
        if tag[0] == "W":
            src.width, have_w = int(tag[1:]), True
        elif tag[0] == "H":
            src.height, have_h = int(tag[1:]), True
        elif tag[0] == "C" and not tag.startswith("C420"):
            raise RuntimeError(f"unsupported Y4M colorspace {tag} (only 4:2:0 accepted)")
    if not (have_w and have_h):
        raise RuntimeError("Y4M header missing W or H tag")
    check_dimensions(src.width, src.height)
    return src


def open_i420(path: str, width: int, height: int) -> SequenceSource:
    check_dimensions(width, height)
    src = SequenceSource(path=path, format=I420, width=width, height=height)
    size = os.path.getsize(path)
    if size % src.frame_bytes():
        raise RuntimeError(f"{path}: size is not a multiple of the I420 frame size")
    src.frame_count = size // src.frame_bytes()
    return src


def open_y4m(path: str) -> SequenceSource:
    with open(path, "rb") as f:
        header = f.readline()
        if not header.endswith(b"\n"):
            raise RuntimeError(f"cannot read Y4M header from {path}")
        src = parse_y4m_header(header[:-1].decode("latin-1"))
        marker = f.readline()
    src.path = path
    src.header_bytes = len(header)
    if not marker:
        raise RuntimeError(f"{path}: Y4M stream has no frames")
    if not marker.startswith(b"FRAME"):
        raise RuntimeError(f"{path}: expected FRAME marker")
    src.frame_marker_bytes = len(marker)
    stride = src.frame_marker_bytes + src.frame_bytes()
    payload = os.path.getsize(path) - src.header_bytes
    if payload % stride:
        raise RuntimeError(f"{path}: truncated or irregular Y4M stream")
    src.frame_count = payload // stride
    return src


def open_sequence(path: str, width: int = 0, height: int = 0) -> SequenceSource:
    """Y4M by extension (``.y4m``), else headerless I420 of the given size."""
    if path.lower().endswith(".y4m"):
        return open_y4m(path)
    return open_i420(path, width, height)


def read_frames(src: SequenceSource, count: Optional[int] = None, chroma: bool = False):
    """Frames 0..count-1 as a ``[count, H, W]`` uint8 luma array (and, with
    ``chroma``, ``[count, 2, H/2, W/2]``), one sequential read of the file."""
    n = src.frame_count if count is None else count
    if n < 0 or n > src.frame_count:
        raise IndexError(f"frame index {n - 1} out of range [0,{src.frame_count})")
    W, H, fb = src.width, src.height, src.frame_bytes()
    stride = fb + (src.frame_marker_bytes if src.format == Y4M else 0)
    raw = np.fromfile(src.path, dtype=np.uint8, count=src.header_bytes + n * stride)
    body = raw[src.header_bytes:].reshape(n, stride) if n else np.zeros((0, stride), np.uint8)
    if src.format == Y4M:
        m = body[:, : src.frame_marker_bytes]
        if n and (not (m[:, :5] == np.frombuffer(b"FRAME", np.uint8)).all() or not (m[:, -1] == 10).all()):
            bad = int(np.flatnonzero(~((m[:, :5] == np.frombuffer(b"FRAME", np.uint8)).all(1) & (m[:, -1] == 10)))[0])
            raise RuntimeError(f"{src.path}: irregular FRAME marker at index {bad}")
        body = body[:, src.frame_marker_bytes:]
    luma = np.ascontiguousarray(body[:, : W * H].reshape(n, H, W))
    if not chroma:
        return luma
    c = np.ascontiguousarray(body[:, W * H:].reshape(n, 2, H // 2, W // 2))
    return luma, c


def pinned_empty(shape) -> np.ndarray:
    """A uint8 array in page-locked host memory (torch's pinned allocator) so
    the host pipeline's H2D copies run asynchronously at full PCIe rate;
    plain memory when torch / CUDA are unavailable."""
    try:
        import torch

        if torch.cuda.is_available():
            return torch.empty(tuple(shape), dtype=torch.uint8, pin_memory=True).numpy()
    except ImportError:
        pass
    return np.empty(tuple(shape), np.uint8)


def stream_frames(src: SequenceSource, count: Optional[int] = None, out: Optional[np.ndarray] = None, first: int = 0) -> np.ndarray:
    """Luma of frames first..first+count-1 read straight into ``out`` (default:
    pinned memory), one ``readinto`` per frame, chroma skipped; Y4M markers
    checked."""
    n = src.frame_count - first if count is None else count
    if first < 0 or n < 0 or first + n > src.frame_count:
        raise IndexError(f"frame index {first + n - 1} out of range [0,{src.frame_count})")
    W, H = src.width, src.height
    out = pinned_empty((n, H, W)) if out is None else out
    if out.shape != (n, H, W) or out.dtype != np.uint8 or not out.flags.c_contiguous:
        raise ValueError("out must be a contiguous uint8 array [frames, H, W]")
    csize = W * H // 2
    stride = W * H * 3 // 2 + (src.frame_marker_bytes if src.format == Y4M else 0)
    with open(src.path, "rb", buffering=0) as f:
        f.seek(src.header_bytes + first * stride)
        for i in range(n):
            if src.format == Y4M:
                m = f.read(src.frame_marker_bytes)
                if len(m) != src.frame_marker_bytes or not m.startswith(b"FRAME") or not m.endswith(b"\n"):
                    raise RuntimeError(f"{src.path}: irregular FRAME marker at index {i}")
            view = memoryview(out[i]).cast("B")
            got = 0
            while got < W * H:
                k = f.readinto(view[got:])
                if not k:
                    raise RuntimeError(f"short read (frame payload) in {src.path}")
                got += k
            f.seek(csize, 1)
    return out


def read_pgm(path: str) -> np.ndarray:
    with open(path, "rb") as f:
        data = f.read()
    if data[:2] != b"P5":
        raise RuntimeError(f"{path}: not a binary P5 PGM")
    pos, vals = 2, []
    for _ in range(3):
        while pos < len(data) and data[pos:pos + 1] in (b" ", b"\t", b"\r", b"\n", b"#"):
            if data[pos:pos + 1] == b"#":
                nl = data.find(b"\n", pos)
                pos = len(data) if nl < 0 else nl + 1
            else:
                pos += 1
        start = pos
        while pos < len(data) and data[pos:pos + 1].isdigit():
            pos += 1
        if start == pos:
            raise RuntimeError(f"malformed PGM header in {path}")
        vals.append(int(data[start:pos]))
    w, h, maxval = vals
    if w <= 0 or h <= 0 or maxval <= 0 or maxval > 255:
        raise RuntimeError(f"{path}: unsupported PGM geometry or maxval")
    pos += 1  # single whitespace byte after maxval
    payload = np.frombuffer(data, dtype=np.uint8, count=min(w * h, max(0, len(data) - pos)), offset=pos)
    if payload.size != w * h:
        raise RuntimeError(f"{path}: truncated PGM payload")
    return payload.reshape(h, w).copy()


def write_gray_pgm(plane: np.ndarray, path: str):  # video_io.cpp:216-223
    h, w = plane.shape
    with open(path, "wb") as f:
        f.write(b"P5\n%d %d\n255\n" % (w, h))
        f.write(np.ascontiguousarray(plane, dtype=np.uint8).tobytes())


def binarize(gray: np.ndarray, threshold: int = 128) -> np.ndarray:  # frame.cpp:50-56
    return np.where(gray >= threshold, 255, 0).astype(np.uint8)


def read_masks(src: MaskSource, count: int, width: int, height: int, out: Optional[np.ndarray] = None, first: int = 0) -> np.ndarray:
    """``[count, H, W]`` binarised masks of frames first.. (read_mask,
    video_io.cpp:184-192)."""
    if not src.present():
        raise RuntimeError("read_mask called without a mask pattern")
    out = np.empty((count, height, width), np.uint8) if out is None else out
    for i in range(count):
        gray = read_pgm(src.path_for(first + i))
        if gray.shape != (height, width):
            raise RuntimeError(f"mask {src.path_for(first + i)} is {gray.shape[1]}x{gray.shape[0]}, video is {width}x{height}")
        out[i] = binarize(gray, src.threshold)
    return out


def estimate_stream(src: SequenceSource, cfg, masks: Optional[MaskSource] = None, chunk: int = 8, device: int = 0):
    """A sequence file through the GPU in chunks of `chunk` frame pairs, I/O
    overlapped with the estimation (pinned streaming I/O): a reader
    thread fills two pinned host slots with chunk k+1's frames (and masks)
    while chunk k crosses PCIe on a copy stream and runs on a compute stream;
    chunk k's frames are [s, s + n + d) (pairs s .. s+n-1), and PA's first pair
    of a chunk takes the previous chunk's last field as its temporal candidates
    (me_b200_run_sequence_prev_dev), so the result equals one whole-sequence
    run (run_experiment's pair loop, bench.cpp:155-205).  Returns (recs
    [pairs, rows, cols], stats [pairs]) in the record / stats dtypes."""
    import ctypes as C
    import queue
    import threading

    import torch

    from . import _lib
    from .api import Algo

    d, bs = cfg.search.ref_distance, cfg.search.block_size
    W, H, F = src.width, src.height, src.frame_count
    pairs = F - d
    if pairs < 1:
        raise ValueError("ref_distance must be smaller than the frame count")
    rows, cols = H // bs, W // bs
    nchunks = (pairs + chunk - 1) // chunk
    dev = torch.device("cuda", device)
    slots = [pinned_empty((2, chunk + d, H, W)) for _ in range(2)]
    dslots = [torch.empty((2, chunk + d, H, W), dtype=torch.uint8, device=dev) for _ in range(2)]
    out_r = torch.empty((pairs, rows, cols, 16), dtype=torch.uint8, pin_memory=True)
    out_s = torch.empty((pairs, 48), dtype=torch.uint8, pin_memory=True)
    recs = torch.empty((2, chunk, rows, cols, 16), dtype=torch.uint8, device=dev)
    stats = torch.empty((2, chunk, 48), dtype=torch.uint8, device=dev)
    prev = torch.zeros((rows * cols, 2), dtype=torch.int32, device=dev)
    copy_st, comp_st = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    free = [threading.Event(), threading.Event()]
    for e in free:
        e.set()
    ready: "queue.Queue" = queue.Queue()

    def reader():
        try:
            for k in range(nchunks):
                s0, n = k * chunk, min(chunk, pairs - k * chunk)
                slot = k & 1
                free[slot].wait()
                free[slot].clear()
                stream_frames(src, n + d, slots[slot][0, : n + d], first=s0)
                if masks is not None and masks.present():
                    read_masks(masks, n + d, W, H, slots[slot][1, : n + d], first=s0)
                ready.put((k, s0, n))
        except Exception as e:  # reported by the consumer
            ready.put(e)

    th = threading.Thread(target=reader, daemon=True)
    th.start()
    c = cfg.c()
    lib = _lib.lib()
    done = [None, None]   # compute of the chunk that last used a device slot
    pending = None        # (copy event, host slot) of the previous chunk
    for _ in range(nchunks):
        item = ready.get()
        if isinstance(item, Exception):
            raise item
        k, s0, n = item
        slot = k & 1
        hs = torch.from_numpy(slots[slot])
        if done[slot] is not None:  # the device slot's previous chunk has been estimated
            copy_st.wait_event(done[slot])
        with torch.cuda.stream(copy_st):
            dslots[slot][:, : n + d].copy_(hs[:, : n + d], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy_st)
        comp_st.wait_event(ev)
        luma, alpha = dslots[slot][0], dslots[slot][1]
        rv, sv = recs[slot], stats[slot]
        _lib.check(lib.me_b200_run_sequence_prev_dev(
            _lib.ctx(device), C.byref(c), n + d, W, H, C.c_void_p(luma.data_ptr()),
            C.c_void_p(alpha.data_ptr()) if masks is not None and masks.present() else None,
            C.c_void_p(prev.data_ptr()) if (k > 0 and cfg.algo == Algo.PA) else None,
            int(not cfg.search.halfpel), C.c_void_p(rv.data_ptr()), C.c_void_p(sv.data_ptr()),
            C.c_void_p(comp_st.cuda_stream)))
        with torch.cuda.stream(comp_st):
            if cfg.algo == Algo.PA:  # the last pair's field: the next chunk's temporal candidates
                prev.copy_(rv[n - 1].reshape(rows * cols, 16).view(torch.int16)[:, 0:2].to(torch.int32))
            out_r[s0: s0 + n].copy_(rv[:n], non_blocking=True)
            out_s[s0: s0 + n].copy_(sv[:n], non_blocking=True)
            done[slot] = torch.cuda.Event()
            done[slot].record(comp_st)
        if pending is not None:  # the previous chunk's host slot may be refilled
            pending[0].synchronize()
            free[pending[1]].set()
        pending = (ev, slot)
    if pending is not None:
        free[pending[1]].set()
    comp_st.synchronize()
    th.join()
    return out_r.numpy().view(_lib.rec_dtype()).reshape(pairs, rows, cols).copy(), out_s.numpy().view(_lib.stats_dtype()).reshape(pairs).copy()


def write_i420(path: str, luma: np.ndarray, chroma: Optional[np.ndarray] = None, y4m: bool = False):
    """Writes frames (gray chroma 128 when absent, append_i420_frame
    video_io.cpp:225-240); ``y4m`` adds the stream header and FRAME markers."""
    n, H, W = luma.shape
    gray = np.full((2, H // 2, W // 2), 128, np.uint8)
    with open(path, "wb") as f:
        if y4m:
            f.write(b"YUV4MPEG2 W%d H%d F25:1 Ip A1:1 C420jpeg\n" % (W, H))
        for i in range(n):
            if y4m:
                f.write(b"FRAME\n")
            f.write(np.ascontiguousarray(luma[i]).tobytes())
            f.write((gray if chroma is None else np.ascontiguousarray(chroma[i])).tobytes())
