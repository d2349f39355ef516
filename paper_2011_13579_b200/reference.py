"""The reference decoder module's API (pkg/src/vitertile/reference.py) on the B200.

``forward_batch`` / ``traceback_batch`` (reference.py:95-144) are the two
stages of the reference decoder with their full outputs -- survivor decisions
(F, N, S), final metrics (F, S), optionally the per-stage metric history --
computed by vt_forward_batch / vt_traceback_batch (csrc/vt_forward.cu) in
exact int64 arithmetic.  ``forward`` / ``traceback`` / ``DecoderState`` wrap
them for one frame (reference.py:147-164), and ``decode_reference`` with
non-uniform initial metrics runs on them.  ``decode_batch``, ``SoftFrame`` and
``decode_reference`` are the package's fused-kernel implementations.
LLRs (and initial metrics) must be integer-valued: int8 quantised LLRs, the
domain on which the B200 decoder is bit-exact (``quantize_llr``).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from ._lib import check, lib
from .codes import CodeSpec
from .decoder import SoftFrame, _as_int8_llr, _code, _ptr, _stream_ptr, _torch, decode_batch, decode_reference

__all__ = ["SoftFrame", "DecoderState", "branch_metric", "forward", "traceback", "decode_reference",
           "decode_batch", "predecessors", "forward_batch", "traceback_batch"]


@dataclass
class DecoderState:
    """Forward-pass output (reference.py:51-57): survivors (N, S) uint8, final
    metrics (S,), metric history (N, S) when requested."""

    survivors: np.ndarray
    final_metrics: np.ndarray
    metric_history: np.ndarray | None = None


def predecessors(state: int, spec: CodeSpec) -> tuple[int, int]:
    """reference.py:60-63: the two predecessors of `state` in tie-rule order."""
    beta = state & (spec.num_butterflies - 1)
    return 2 * beta, 2 * beta + 1


def branch_metric(branch_bits, llr_t) -> float:
    """reference.py:85-92: correlation of a branch output with one stage's LLRs."""
    bits = np.asarray(branch_bits, dtype=np.float64)
    llr = np.asarray(llr_t, dtype=np.float64)
    if bits.shape != llr.shape:
        raise ValueError("branch output and LLR lengths differ")
    return float(np.sum((1.0 - 2.0 * bits) * llr))


def _int_metrics(initial_metrics, f: int, s: int) -> tuple[np.ndarray, int]:
    init = np.asarray(initial_metrics, dtype=np.float64)
    if not np.all(np.isfinite(init)) or np.any(init != np.rint(init)):
        raise ValueError("initial metrics must be integer-valued (the B200 decoder is exact in int64)")
    if init.ndim <= 1:
        return np.ascontiguousarray(np.broadcast_to(init, (s,)), dtype=np.int64), 0
    return np.ascontiguousarray(np.broadcast_to(init, (f, s)), dtype=np.int64), 1


def forward_batch(llrs, spec: CodeSpec, initial_metrics=None, renormalize: bool = False,
                  keep_history: bool = False):
    """reference.forward_batch: llrs (F, B, N) -> (survivors (F, N, S) uint8, final
    metrics (F, S) float64, metric history (F, N, S) float64 or None)."""
    torch = _torch()
    arr = np.asarray(llrs)
    if arr.ndim != 3 or arr.shape[1] != spec.outputs_per_bit:
        raise ValueError("LLR batch must have shape (F, B, N)")
    f, b, n = arr.shape
    s = spec.num_states
    q = np.ascontiguousarray(np.transpose(_as_int8_llr(arr), (0, 2, 1)))  # (F, N, B)
    dev = torch.device("cuda", torch.cuda.current_device())
    d_llr = torch.from_numpy(q).to(dev)
    surv = torch.empty((f, n, s), dtype=torch.uint8, device=dev)
    lam = torch.empty((f, s), dtype=torch.int64, device=dev)
    hist = torch.empty((f, n, s), dtype=torch.int64, device=dev) if keep_history else None
    init_t, per_frame = None, 0
    if initial_metrics is not None:
        init, per_frame = _int_metrics(initial_metrics, f, s)
        init_t = torch.from_numpy(init).to(dev)
    check(lib().vt_forward_batch(ctypes.byref(_code(spec)), _ptr(d_llr), f, n, _ptr(init_t), per_frame,
                                 1 if renormalize else 0, _ptr(surv), _ptr(lam), _ptr(hist), _stream_ptr(None)))
    return (surv.cpu().numpy(), lam.cpu().numpy().astype(np.float64),
            hist.cpu().numpy().astype(np.float64) if hist is not None else None)


def traceback_batch(survivors, final_metrics, spec: CodeSpec) -> np.ndarray:
    """reference.traceback_batch: (F, N, S) survivors + (F, S) final metrics -> bits (F, N)."""
    torch = _torch()
    sv = np.ascontiguousarray(np.asarray(survivors), dtype=np.uint8)
    lm = np.asarray(final_metrics, dtype=np.float64)
    if sv.ndim != 3 or lm.shape != (sv.shape[0], sv.shape[2]) or sv.shape[2] != spec.num_states:
        raise ValueError("survivors must be (F, N, S) and final metrics (F, S)")
    if np.any(lm != np.rint(lm)):
        raise ValueError("final metrics must be integer-valued")
    f, n, _ = sv.shape
    dev = torch.device("cuda", torch.cuda.current_device())
    d_sv = torch.from_numpy(sv).to(dev)
    d_lm = torch.from_numpy(np.ascontiguousarray(lm, dtype=np.int64)).to(dev)
    bits = torch.empty((f, n), dtype=torch.uint8, device=dev)
    check(lib().vt_traceback_batch(ctypes.byref(_code(spec)), _ptr(d_sv), _ptr(d_lm), f, n, _ptr(bits),
                                   _stream_ptr(None)))
    return bits.cpu().numpy()


def forward(frame, spec: CodeSpec, initial_metrics=None, renormalize: bool = False,
            keep_history: bool = False) -> DecoderState:
    """reference.forward (reference.py:147-158): one (B, N) frame."""
    llr = frame.llr if isinstance(frame, SoftFrame) else np.asarray(frame, dtype=np.float64)
    surv, lam, hist = forward_batch(llr[None, :, :], spec, initial_metrics, renormalize, keep_history)
    return DecoderState(surv[0], lam[0], hist[0] if hist is not None else None)


def traceback(state: DecoderState, spec: CodeSpec) -> np.ndarray:
    """reference.traceback (reference.py:161-164)."""
    return traceback_batch(state.survivors[None, :, :], state.final_metrics[None, :], spec)[0]
