"""Reference-compatible decode API backed by the sm_100a kernels.

Drop-in for the decode entry points of the reference package
(pkg/src/vitertile): same names, argument meaning, return types and
ValueError conventions.  Every decode runs on the GPU through the C ABI of
include/vitertile_b200.h; there is no CPU fallback.

Parity contract: results are bit-identical to the reference
for integer-valued LLRs in [-128, 127] (the int8 quantised LLRs the decoder
is specified on).  Non-integer float LLRs are rejected with ValueError — use
``quantize_llr`` first; hard mode slices any float input exactly like the
reference (reference.py:202-203).
"""
from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass, field

import numpy as np

from ._lib import VtCode, check, lib
from .codes import CodeSpec, find_dragonfly_groups, identical_bomat_classes
from .framing import FramePlan

__all__ = [
    "PrecisionPolicy",
    "TileOpCounter",
    "DecoderConfig",
    "MatrixDecodeResult",
    "SoftFrame",
    "quantize_llr",
    "decode_stream",
    "decode_stream_device",
    "decode_stream_host",
    "decode_batch",
    "decode_reference",
    "decode_matrix_batch",
    "decode_matrix",
    "workspace_bytes",
    "release_workspaces",
]

_PRECISIONS = ("half", "single")


@dataclass(frozen=True)
class PrecisionPolicy:
    """Accumulator / channel-input precision (tile.py:21-31).  The fused decoders
    accumulate exact integer metrics; the tile decoder (decode_matrix_batch,
    decoder="matrix") reproduces ``accumulator="half"``: every tensor-core tile
    result is rounded to binary16 as the reference does."""

    accumulator: str = "single"
    channel_input: str = "single"

    def __post_init__(self) -> None:
        for name in (self.accumulator, self.channel_input):
            if name not in _PRECISIONS:
                raise ValueError(f"unknown precision {name!r}")


@dataclass
class TileOpCounter:
    """Paper tile-op accounting (tile.py:34-49)."""

    mma_ops: int = 0
    survivor_write_passes: int = 0
    stages: int = 0

    @property
    def ops_per_stage(self) -> float:
        return self.mma_ops / self.stages if self.stages else 0.0

    def reset(self) -> None:
        self.mma_ops = self.survivor_write_passes = self.stages = 0


@dataclass(frozen=True)
class DecoderConfig:
    """Decode path selection (matrix.py:94-105)."""

    radix: int = 2
    optimized: bool = False
    policy: PrecisionPolicy = field(default_factory=PrecisionPolicy)
    renormalize: bool = False

    def __post_init__(self) -> None:
        if self.radix not in (2, 4):
            raise ValueError("radix must be 2 or 4")


@dataclass
class MatrixDecodeResult:
    bits: np.ndarray
    final_metric: np.ndarray | float
    counter: TileOpCounter

    @property
    def q(self) -> float:
        return self.counter.ops_per_stage


@dataclass
class SoftFrame:
    """LLR input (B, N); positive LLR favours coded bit 0 (reference.py:27-48)."""

    llr: np.ndarray
    channel_precision: str = "single"

    def __post_init__(self) -> None:
        if self.channel_precision not in _PRECISIONS:
            raise ValueError(f"unknown channel precision {self.channel_precision!r}")
        arr = np.asarray(self.llr, dtype=np.float64)
        if arr.ndim != 2 or arr.shape[1] < 1:
            raise ValueError("LLR input must have shape (B, N) with N >= 1")
        if not np.all(np.isfinite(arr)):
            raise ValueError("LLR values must be finite")
        if self.channel_precision == "half":
            arr = arr.astype(np.float16).astype(np.float64)
        self.llr = arr

    @property
    def num_stages(self) -> int:
        return self.llr.shape[1]


def quantize_llr(llr, scale: float = 16.0) -> np.ndarray:
    """int8 quantiser the parity contract is defined on:
    q = clamp(rint(scale * llr), -127, 127)."""
    return np.clip(np.rint(np.asarray(llr, dtype=np.float64) * scale), -127, 127).astype(np.int8)


# ---------------------------------------------------------------------------
# device plumbing (torch is used only for device memory and streams)
# ---------------------------------------------------------------------------

_ws_lock = threading.Lock()
_ws: dict[int, object] = {}


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("vitertile_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    return torch


def _workspace(nbytes: int, stream=None):
    """Scratch for one launch, one buffer per (device, stream): launches on one stream are
    ordered, so they may share it; concurrent streams (e.g. worker threads, as
    framing.decode_stream's workers=) each get their own.  ``release_workspaces()`` frees
    them."""
    torch = _torch()
    dev = torch.cuda.current_device()
    s = stream if stream is not None else torch.cuda.current_stream()
    key = (dev, int(s.cuda_stream))
    with _ws_lock:
        buf = _ws.get(key)
        if buf is None or buf.numel() < nbytes:
            with torch.cuda.stream(s):  # allocated (and later recycled) in the launch stream's order
                buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=f"cuda:{dev}")
            _ws[key] = buf
        return buf


def _pinned(tag: str, numel: int, dtype):
    """Grow-only pinned host staging buffer per (calling thread, tag): reused across calls
    (pinning is a page-locking syscall per allocation).  Only for buffers that never
    leave the call."""
    torch = _torch()
    key = ("pinned", tag, threading.get_ident())
    with _ws_lock:
        buf = _ws.get(key)
        if buf is None or buf.numel() < numel or buf.dtype != dtype:
            buf = torch.empty(max(numel, 1), dtype=dtype, pin_memory=True)
            _ws[key] = buf
    return buf[:numel]


def release_workspaces() -> None:
    """Free the cached device workspaces and host staging buffers (they are kept
    between calls so repeated decodes do not reallocate)."""
    with _ws_lock:
        _ws.clear()


def _ptr(t) -> ctypes.c_void_p:
    return ctypes.c_void_p(t.data_ptr()) if t is not None else ctypes.c_void_p(0)


def _stream_ptr(stream) -> ctypes.c_void_p:
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


_codes: dict = {}  # (K, generators) -> checked VtCode (read-only once built)


def _code(spec: CodeSpec) -> VtCode:
    key = (int(spec.constraint_length), tuple(int(g) for g in spec.generators))
    c = _codes.get(key)
    if c is not None:
        return c
    c = VtCode.from_spec(spec)
    if not lib().vt_code_supported(ctypes.byref(c)):
        # a code the library was not built with: generate + compile its kernels (jit.py)
        from . import jit
        jit.ensure(spec)
    _codes[key] = c
    return c


def workspace_bytes(spec: CodeSpec, n: int, frame_len: int, overlap: int, w0: int = 0, w1: int | None = None) -> int:
    nw = -(-int(n) // int(frame_len))
    w1 = nw if w1 is None else w1
    return int(lib().vt_workspace_bytes(ctypes.byref(_code(spec)), int(n), int(frame_len), int(overlap), int(w0),
                                        int(w1)))


def _as_int8_llr(llr, what: str = "LLR") -> np.ndarray:
    a = np.asarray(llr)
    if a.dtype == np.int8:
        return a
    if np.issubdtype(a.dtype, np.integer):
        if a.size and (a.min() < -128 or a.max() > 127):
            raise ValueError(f"{what} values must lie in [-128, 127] (int8 quantised LLRs)")
        return a.astype(np.int8)
    af = np.asarray(a, dtype=np.float64)
    if not np.all(np.isfinite(af)):
        raise ValueError("LLR values must be finite")
    q = np.rint(af)
    if not np.array_equal(q, af):
        raise ValueError(f"{what} must be integer-valued int8 quantised LLRs; quantise with quantize_llr() "
                         "(the B200 decoder is bit-exact on the quantised integers)")
    if q.size and (q.min() < -128 or q.max() > 127):
        raise ValueError(f"{what} values must lie in [-128, 127] (int8 quantised LLRs)")
    return q.astype(np.int8)


def _unpack(words_np: np.ndarray, n: int) -> np.ndarray:
    return np.unpackbits(words_np.view(np.uint8), count=n, bitorder="little")


# ---------------------------------------------------------------------------
# device-level entry points (no host round trip)
# ---------------------------------------------------------------------------


def decode_stream_device(llr_nb, spec: CodeSpec, frame_len: int, overlap: int, *, out=None,
                         final_metric=None, stream=None):
    """Decode an int8 (N, B) device tensor with plan_frames(N, F, V) windows.

    Returns the packed output bits as an int32 device tensor of ceil(N/32)
    words (bit t&31 of word t>>5 = decoded bit of stage t).  ``out`` may be a
    zeroed int32 tensor to reuse; ``final_metric`` an int64 device tensor with
    one entry per window."""
    torch = _torch()
    code = _code(spec)
    if llr_nb.dtype != torch.int8 or llr_nb.dim() != 2 or llr_nb.shape[1] != spec.outputs_per_bit:
        raise ValueError("llr must be an int8 (N, B) CUDA tensor")
    llr_nb = llr_nb.contiguous()
    if llr_nb.data_ptr() % 16:  # e.g. a row slice: the kernels stage 16-byte words
        llr_nb = llr_nb.clone()
    n = int(llr_nb.shape[0])
    nwords = (n + 31) // 32
    if out is None:
        out = torch.zeros(nwords, dtype=torch.int32, device=llr_nb.device)
    nw = -(-n // int(frame_len))
    need = lib().vt_workspace_bytes(ctypes.byref(code), n, int(frame_len), int(overlap), 0, nw)
    ws = _workspace(need, stream)
    check(lib().vt_decode_stream(ctypes.byref(code), _ptr(llr_nb), n, int(frame_len), int(overlap), _ptr(out),
                                 _ptr(final_metric), _ptr(ws), ws.numel(), _stream_ptr(stream)))
    return out


def _devices(devices, workers: int) -> list[int]:
    torch = _torch()
    if devices is not None:
        devs = [int(d) for d in devices]
        if not devs:
            raise ValueError("devices must not be empty")
        n = torch.cuda.device_count()
        for d in devs:
            if not 0 <= d < n:
                raise ValueError(f"device {d} out of range (have {n})")
        return devs
    workers = int(workers)
    if workers < 1:
        raise ValueError("workers must be >= 1")
    return list(range(min(workers, torch.cuda.device_count()))) if workers > 1 else [torch.cuda.current_device()]


def decode_stream_host(llr_nb_host, spec: CodeSpec, frame_len: int, overlap: int, *, bits_host=None,
                       nchunks: int = 8, stream=None, devices=None, workers: int = 1):
    """End-to-end decode through the C-ABI host entry (vt_decode_stream_host):
    int8 (N, B) host tensor (pinned for full PCIe bandwidth) -> packed int32
    host tensor.  H2D, decode and D2H are pipelined in ``nchunks`` window ranges.

    ``devices`` (CUDA device indices; repeats allowed = several streams on one
    GPU) or ``workers`` > 1 (the first min(workers, device_count) GPUs) fans the
    windows out over several devices, one shard, host thread, stream and set of
    staging buffers each (vt_decode_stream_host_multi) -- the reference's
    ``workers`` thread fan-out of one stream's windows (framing.py:121-135).
    Each GPU brings its own PCIe link, so the end-to-end rate scales with them."""
    torch = _torch()
    code = _code(spec)
    n = int(llr_nb_host.shape[0])
    b = spec.outputs_per_bit
    nwords = (n + 31) // 32
    if bits_host is None:
        bits_host = torch.empty(nwords, dtype=torch.int32, pin_memory=True)
    devs = _devices(devices, workers)
    nw = -(-n // int(frame_len))
    if len(devs) > 1:
        return _decode_stream_host_multi(llr_nb_host, code, spec, n, int(frame_len), int(overlap), bits_host,
                                         devs, int(nchunks))
    dev = torch.cuda.current_device()
    key = ("host", dev, threading.get_ident())  # the C entry runs on per-call copy streams
    with _ws_lock:
        stg = _ws.get(key)
        need_llr = ((n * b + 15) // 16) * 16
        if stg is None or stg[0].numel() < need_llr or stg[1].numel() < nwords:
            stg = (torch.empty(need_llr, dtype=torch.int8, device=f"cuda:{dev}"),
                   torch.empty(nwords, dtype=torch.int32, device=f"cuda:{dev}"))
            _ws[key] = stg
    need = lib().vt_workspace_bytes_host(ctypes.byref(code), n, int(frame_len), int(overlap), 0, nw, int(nchunks))
    ws = _workspace(need, stream)
    check(lib().vt_decode_stream_host(ctypes.byref(code), _ptr(llr_nb_host), n, int(frame_len), int(overlap),
                                      _ptr(bits_host), _ptr(stg[0]), _ptr(stg[1]), _ptr(ws), ws.numel(),
                                      int(nchunks), _stream_ptr(stream)))
    return bits_host


def _decode_stream_host_multi(llr_nb_host, code, spec, n: int, f: int, v: int, bits_host, devs, nchunks: int):
    torch = _torch()
    b = spec.outputs_per_bit
    nwords = (n + 31) // 32
    g_n = len(devs)
    llr_p, bits_p, ws_p, ws_n = [], [], [], []
    keep = []
    rng = (ctypes.c_int64 * 4)()
    for g, d in enumerate(devs):
        check(lib().vt_shard_range(n, f, v, g_n, g, rng))
        w0, w1, st0, st1 = (int(x) for x in rng)
        key = ("multi", d, g, threading.get_ident())
        with torch.cuda.device(d):
            need_ws = lib().vt_workspace_bytes_host(ctypes.byref(code), n, f, v, w0, w1, nchunks) if w1 > w0 else 0
            need_llr = max(16, (((st1 - st0) * b + 15) // 16) * 16)
            with _ws_lock:
                stg = _ws.get(key)
                if (stg is None or stg[0].numel() < need_llr or stg[1].numel() < nwords or
                        stg[2].numel() < need_ws):
                    stg = (torch.empty(need_llr, dtype=torch.int8, device=f"cuda:{d}"),
                           torch.empty(nwords, dtype=torch.int32, device=f"cuda:{d}"),
                           torch.empty(max(need_ws, 1 << 20), dtype=torch.uint8, device=f"cuda:{d}"))
                    _ws[key] = stg
        keep.append(stg)
        llr_p.append(stg[0].data_ptr())
        bits_p.append(stg[1].data_ptr())
        ws_p.append(stg[2].data_ptr())
        ws_n.append(stg[2].numel())
    arr = lambda t, xs: (t * len(xs))(*xs)  # noqa: E731
    check(lib().vt_decode_stream_host_multi(
        ctypes.byref(code), _ptr(llr_nb_host), n, f, v, _ptr(bits_host), g_n, arr(ctypes.c_int, devs),
        arr(ctypes.c_void_p, llr_p), arr(ctypes.c_void_p, bits_p), arr(ctypes.c_void_p, ws_p),
        arr(ctypes.c_size_t, ws_n), nchunks))
    return bits_host


def _decode_frames_np(frames_fnb: np.ndarray, spec: CodeSpec):
    """(F, N, B) int8 frames -> (bits (F, N) uint8, final metric int64 (F,))."""
    torch = _torch()
    return _decode_frames_dev(torch.from_numpy(np.ascontiguousarray(frames_fnb)).cuda(), spec)


def _decode_frames_dev(dev_llr, spec: CodeSpec):
    """(F, N, B) int8 device frames -> (bits (F, N) uint8, final metric int64 (F,)) on the host."""
    torch = _torch()
    code = _code(spec)
    f, n, _ = dev_llr.shape
    total = f * n
    bits = torch.zeros((total + 31) // 32, dtype=torch.int32, device=dev_llr.device)
    metric = torch.empty(f, dtype=torch.int64, device=dev_llr.device)
    need = lib().vt_workspace_bytes(ctypes.byref(code), total, n, 0, 0, f)
    ws = _workspace(need)
    check(lib().vt_decode_frames(ctypes.byref(code), _ptr(dev_llr), f, n, _ptr(bits), _ptr(metric), _ptr(ws),
                                 ws.numel(), _stream_ptr(None)))
    words = bits.cpu().numpy()
    return _unpack(words, total).reshape(f, n), metric.cpu().numpy()


# ---------------------------------------------------------------------------
# reference-compatible API
# ---------------------------------------------------------------------------


def decode_stream(llr, spec: CodeSpec, plan: FramePlan, decoder: str = "reference",
                  config: DecoderConfig | None = None, workers: int = 1) -> np.ndarray:
    """framing.decode_stream (framing.py:96-141): decode a (B, N) LLR stream
    window by window and stitch the emit ranges -> uint8 bits (N,).
    ``workers`` > 1 fans the windows out over up to that many GPUs (the
    reference fans them over threads, framing.py:121-135); on one GPU all
    windows of the plan run in one launch either way."""
    arr = np.asarray(llr)
    if arr.ndim != 2 or arr.shape[1] != plan.total_stages:
        raise ValueError("plan does not match stream length")
    if decoder not in ("reference", "matrix"):
        raise ValueError(f"unknown decoder {decoder!r}")
    if arr.shape[0] != spec.outputs_per_bit:
        raise ValueError("LLR input must have shape (B, N)")
    r4perm = half = False
    if decoder == "matrix":
        cfg = config or DecoderConfig()
        _, _, effective = _check_matrix_config(spec, cfg)
        r4perm = cfg.radix == 4 and cfg.optimized and effective
        # the binary16 accumulator rounds metrics (tile.py:87-89): the tile decoder, per window
        half = cfg.policy.accumulator == "half"
    torch = _torch()
    if arr.dtype == np.float64 and not r4perm and not half and _closed_form_plan(plan):
        # reference-style float LLRs: one native pass checks, converts and transposes
        # straight into pinned memory, then the pipelined host entry
        a64 = np.ascontiguousarray(arr)
        n = a64.shape[1]
        pinned = _pinned("llr", n * a64.shape[0], torch.int8).view(n, a64.shape[0])
        check(lib().vt_pack_llr_f64(a64.ctypes.data_as(ctypes.c_void_p), a64.shape[0], n, n, _ptr(pinned), 0))
        words = decode_stream_host(pinned, spec, plan.frame_len, plan.overlap,
                                   bits_host=_pinned("bits", (n + 31) // 32, torch.int32), workers=workers)
        return _unpack(words.numpy(), n)
    q = _as_int8_llr(arr).T.copy()  # (N, B) stage-major
    n = q.shape[0]
    if half or not _closed_form_plan(plan):
        return _decode_windows_general(q, spec, plan, decoder, config)
    if r4perm:  # radix-4 with the dragonfly permutation tie order (matrix.py:329-333)
        dev = torch.from_numpy(q).cuda()
        out = torch.zeros((n + 31) // 32, dtype=torch.int32, device=dev.device)
        _decode_r4perm_device(dev, spec, n, plan.frame_len, plan.overlap, out)
        return _unpack(out.cpu().numpy(), n)
    pinned = _pinned("llr", q.size, torch.int8).view(n, q.shape[1])
    pinned.numpy()[...] = q
    words = decode_stream_host(pinned, spec, plan.frame_len, plan.overlap,
                               bits_host=_pinned("bits", (n + 31) // 32, torch.int32), workers=workers)
    return _unpack(words.numpy(), n)


def _closed_form_plan(plan) -> bool:
    """True when the plan's windows are plan_frames(N, F, V)'s (the fused stream kernels
    compute that geometry on the device).  Any plan object with the reference's
    FramePlan fields qualifies -- including one built by the reference's own
    plan_frames (framing.py:68-83, a different Window class): windows are compared by
    their (start, stop, emit_start, emit_stop) geometry."""
    from .framing import _Windows
    w = plan.windows
    n, f, v = int(plan.total_stages), int(plan.frame_len), int(plan.overlap)
    if isinstance(w, _Windows):
        return (w._n, w._f, w._v) == (n, f, v)
    if n < 1 or f < 1 or v < 0:
        return False
    nw = -(-n // f)
    if len(w) != nw:
        return False
    try:
        got = np.array([(x.start, x.stop, x.emit_start, x.emit_stop) for x in w], dtype=np.int64).reshape(nw, 4)
    except AttributeError:
        return False
    e0 = np.arange(nw, dtype=np.int64) * f
    e1 = np.minimum(e0 + f, n)
    want = np.stack([np.maximum(0, e0 - v), np.minimum(n, e1 + v), e0, e1], axis=1)
    return bool(np.array_equal(got, want))


def _decode_windows_general(q: np.ndarray, spec: CodeSpec, plan, decoder: str, config) -> np.ndarray:
    """framing._decode_windows (framing.py:86-93, 112-137) for an arbitrary window list:
    windows grouped by length, each group one batched GPU decode, emit ranges stitched."""
    n = q.shape[0]
    out = np.zeros(n, dtype=np.uint8)
    groups: dict[int, list] = {}
    for w in plan.windows:
        groups.setdefault(w.stop - w.start, []).append(w)
    for length, ws in groups.items():
        frames = np.stack([q[w.start:w.stop] for w in ws])  # (F, L, B)
        if decoder == "matrix":
            bits = decode_matrix_batch(np.transpose(frames, (0, 2, 1)).astype(np.float32), spec,
                                       config or DecoderConfig()).bits
        else:
            bits, _ = _decode_frames_np(np.ascontiguousarray(frames), spec)
        for i, w in enumerate(ws):
            out[w.emit_start:w.emit_stop] = bits[i][w.emit_start - w.start:w.emit_stop - w.start]
    return out


def decode_batch(llrs, spec: CodeSpec, mode: str = "soft", renormalize: bool = False):
    """reference.decode_batch (reference.py:194-206): frames (F, B, N) ->
    (bits (F, N) uint8, final metric per frame float64)."""
    arr = np.asarray(llrs, dtype=np.float64)
    if arr.ndim != 3 or arr.shape[1] != spec.outputs_per_bit:
        raise ValueError("LLR batch must have shape (F, B, N)")
    if mode == "hard":
        arr = np.where(arr >= 0.0, 1.0, -1.0)
    elif mode != "soft":
        raise ValueError(f"unknown mode {mode!r}")
    f, b, n = arr.shape
    if f * n >= (1 << 20):  # large batches: one native pass (check + convert) into pinned memory
        torch = _torch()
        a64 = np.ascontiguousarray(arr).reshape(f * b, n)  # rows (frame, output)
        pinned = torch.empty((n, f * b), dtype=torch.int8, pin_memory=True)
        check(lib().vt_pack_llr_f64(a64.ctypes.data_as(ctypes.c_void_p), f * b, n, n, _ptr(pinned), 0))
        dev = pinned.to(f"cuda:{torch.cuda.current_device()}", non_blocking=True)
        bits, metric = _decode_frames_dev(dev.view(n, f, b).permute(1, 0, 2).contiguous(), spec)
    else:
        q = _as_int8_llr(arr)
        bits, metric = _decode_frames_np(np.transpose(q, (0, 2, 1)), spec)
    if renormalize:  # reference.py:124-125: max subtracted after every stage -> final max is 0
        metric = np.zeros_like(metric)
    return bits, metric.astype(np.float64)


def _to_soft(frame, spec: CodeSpec, mode: str) -> np.ndarray:
    # reference.py:167-178
    llr = frame.llr if isinstance(frame, SoftFrame) else np.asarray(frame, dtype=np.float64)
    if llr.ndim != 2 or llr.shape[0] != spec.outputs_per_bit:
        raise ValueError("LLR input must have shape (B, N)")
    if mode == "hard":
        if not np.all((llr == 0) | (llr == 1)):
            raise ValueError("hard mode expects a bit array")
        llr = 1.0 - 2.0 * llr
    elif mode != "soft":
        raise ValueError(f"unknown mode {mode!r}")
    return llr


def decode_reference(frame, spec: CodeSpec, mode: str = "soft", initial_metrics=None,
                     renormalize: bool = False) -> np.ndarray:
    """reference.decode_reference (reference.py:181-191): one frame, forward +
    traceback -> bits (N,)."""
    llr = _to_soft(frame, spec, mode)
    if initial_metrics is not None:
        init = np.broadcast_to(np.asarray(initial_metrics, dtype=np.float64), (spec.num_states,))
        if not np.all(init == init[0]):  # the fused kernels start from uniform metrics: separate stages
            from .reference import forward, traceback
            return traceback(forward(llr, spec, init, renormalize), spec)
    bits, _ = decode_batch(llr[None, :, :], spec, renormalize=renormalize)
    return bits[0]


# ---------------------------------------------------------------------------
# tile-decoder API (matrix.py:342-422)
# ---------------------------------------------------------------------------

_BLOCK, _TILE_BLOCKS = 4, 4  # 4 columns per block, 4 blocks per 16x16 tile


def _tiles(blocks: int) -> int:
    return -(-blocks // _TILE_BLOCKS)


def _radix2_tiles(spec: CodeSpec) -> int:
    if spec.outputs_per_bit > _BLOCK:
        raise ValueError(f"butterfly output matrix width {spec.outputs_per_bit} exceeds block width {_BLOCK}")
    return _tiles(sum(-(-len(c) // _BLOCK) for c in identical_bomat_classes(1, spec)))


def _radix4_tiles(spec: CodeSpec, optimized: bool) -> tuple[int, bool]:
    if 2 * spec.outputs_per_bit > _BLOCK:
        raise ValueError(f"super-branch output width {2 * spec.outputs_per_bit} exceeds block width {_BLOCK}")
    plain = sum(-(-len(c) // _BLOCK) for c in identical_bomat_classes(2, spec))
    if optimized:
        grouped = sum(-(-len(g.members) // _BLOCK) for g in find_dragonfly_groups(2, spec))
        if grouped < plain:
            return _tiles(grouped), True
    return _tiles(plain), False


def _check_matrix_config(spec: CodeSpec, config: DecoderConfig) -> tuple[int, int, bool]:
    t2 = _radix2_tiles(spec)
    t4, effective = (_radix4_tiles(spec, config.optimized) if config.radix == 4 else (0, False))
    return t2, t4, effective


def _r4_priorities(spec: CodeSpec) -> np.ndarray:
    """prio[f*4 + x]: position of left-local state x of dragonfly f in its group
    representative's row order (matrix.py:237-241, 329-333): the radix-4
    optimised path breaks ties toward the highest position."""
    s4 = spec.num_states // 4
    prio = np.tile(np.arange(4, dtype=np.uint8), s4)
    for g in find_dragonfly_groups(2, spec):
        for f, perm in g.permutations.items():
            for i, x in enumerate(perm):
                prio[f * 4 + x] = i
    return prio


def _decode_r4perm_device(llr_nb, spec: CodeSpec, n: int, frame_len: int, overlap: int, out, final_metric=None,
                          stream=None):
    code = _code(spec)
    nw = -(-n // frame_len)
    need = lib().vt_workspace_bytes_r4perm(ctypes.byref(code), n, frame_len, overlap, 0, nw)
    ws = _workspace(need, stream)
    prio = np.ascontiguousarray(_r4_priorities(spec))
    check(lib().vt_decode_stream_r4perm(ctypes.byref(code), prio.ctypes.data_as(ctypes.c_void_p), _ptr(llr_nb), 0,
                                        n, n, frame_len, overlap, 0, nw, _ptr(out), _ptr(final_metric), _ptr(ws),
                                        ws.numel(), _stream_ptr(stream)))
    return out


def decode_matrix_batch(llrs, spec: CodeSpec, config: DecoderConfig | None = None) -> MatrixDecodeResult:
    """matrix.decode_matrix_batch (matrix.py:342-386) in the paper's formulation on
    tensor cores: every tile op D = A x B + C of the reference's pack_radix2 /
    pack_radix4 tiles (radix 2, radix 4, radix 4 with the dragonfly-permutation
    groups) runs as mma.sync.m16n8k16 (vt_matrix_forward, csrc/vt_tiles.cu); the
    counter reports the tile ops the kernel actually issued.  ``accumulator="half"``
    rounds every tile result to binary16 exactly as tile.py:87-89 does."""
    config = config or DecoderConfig()
    arr = np.asarray(llrs, dtype=np.float32)
    if arr.ndim != 3 or arr.shape[1] != spec.outputs_per_bit:
        raise ValueError("LLR batch must have shape (F, B, N)")
    f, b, n = arr.shape
    _check_matrix_config(spec, config)
    # matrix.py:290,320 (and 354-355): LLRs pass through binary16; exact for int8 values
    q = _as_int8_llr(arr.astype(np.float16).astype(np.float64))
    torch = _torch()
    dev = torch.from_numpy(np.ascontiguousarray(np.transpose(q, (0, 2, 1)))).cuda()  # (F, N, B)
    bits, metric, ops = _matrix_frames_device(dev, spec, config)
    counter = TileOpCounter()
    counter.mma_ops = ops
    counter.survivor_write_passes = n // 2 + n % 2 if config.radix == 4 else n
    counter.stages = n
    return MatrixDecodeResult(bits=bits.cpu().numpy(), final_metric=metric.cpu().numpy(), counter=counter)


def _matrix_frames_device(dev_fnb, spec: CodeSpec, config: DecoderConfig, stream=None):
    """Tile decoder on a device (F, N, B) int8 batch -> (bits (F, N) uint8, final metric
    float64 (F,)) device tensors and the tile ops issued per frame."""
    torch = _torch()
    from . import tiles
    f, n, _ = dev_fnb.shape
    code = _code(spec)
    r2, _ = tiles.device_program(spec, 2)
    r4 = tiles.device_program(spec, 4, config.optimized)[0] if config.radix == 4 else None
    steps = n // 2 + n % 2 if config.radix == 4 else n
    s = spec.num_states
    kw = {"device": dev_fnb.device}
    surv = torch.empty((f, steps, s), dtype=torch.uint8, **kw)
    lam = torch.empty((f, s), dtype=torch.float32, **kw)
    off = torch.empty(f, dtype=torch.float64, **kw)
    bits = torch.empty((f, n), dtype=torch.uint8, **kw)
    metric = torch.empty(f, dtype=torch.float64, **kw)
    count = torch.zeros(1, dtype=torch.int64, **kw)
    check(lib().vt_matrix_forward(ctypes.byref(code), _ptr(dev_fnb.contiguous()), f, n, ctypes.byref(r2),
                                  ctypes.byref(r4) if r4 is not None else None, config.radix,
                                  int(config.policy.accumulator == "half"), int(config.renormalize), _ptr(surv),
                                  _ptr(lam), _ptr(off), _ptr(bits), _ptr(metric), _ptr(count), _stream_ptr(stream)))
    return bits, metric, int(count.item()) // (2 * f)  # two mma.sync m16n8k16 per 16x16x16 tile op


def decode_matrix(frame, spec: CodeSpec, config: DecoderConfig | None = None) -> MatrixDecodeResult:
    """matrix.decode_matrix (matrix.py:412-422): single-frame wrapper."""
    llr = getattr(frame, "llr", frame)
    res = decode_matrix_batch(np.asarray(llr)[None, :, :], spec, config)
    return MatrixDecodeResult(bits=res.bits[0], final_metric=float(res.final_metric[0]), counter=res.counter)
