"""On-disk formats of the reference CLI and a streaming file decoder.

Formats (pkg/src/vitertile/cli.py:4-8, 31-62):
  * bit files: 8-byte little-endian bit count, then the bits packed into
    little-endian bytes, LSB = earliest bit, padded to whole 32-bit words
    (write_bit_file / read_bit_file, cli.py:31-52);
  * LLR files: stage-major, polynomial-minor binary16 ("half") or binary32
    ("single") little-endian scalars (write_llr_file / read_llr_file,
    cli.py:55-62);
  * decoded output of ``vitertile decode``: the decoded bits packed
    little-endian with no header, refused unless the count is byte aligned
    (cli.py:170-173).

The decoder's packed output words (bit t&31 of word t>>5) are exactly the
little-endian byte stream of these files, so decoded bits go from the device
to disk without unpacking.  ``decode_llr_file`` streams an LLR file of any
length through pinned host memory in window-aligned pieces (each piece a
vt_decode_stream_range launch on a stage sub-buffer with its V-stage halo),
so the file never has to fit in host or device memory as float or int8
arrays.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from ._lib import check, lib
from .codes import CodeSpec
from .decoder import _code, _ptr, _stream_ptr, _torch, _workspace

_LLR_DTYPES = {"half": "<f2", "single": "<f4"}


def _llr_np_dtype(dtype: str) -> str:
    try:
        return _LLR_DTYPES[dtype]
    except KeyError:
        raise ValueError(f"LLR dtype must be 'half' or 'single', got {dtype!r}") from None


def write_bit_file(bits, path: str) -> None:
    """cli.write_bit_file (cli.py:31-39): count header + LSB-first packed bits, 4-byte padded."""
    bits = np.asarray(bits, dtype=np.uint8).reshape(-1)
    packed = np.packbits(bits, bitorder="little")
    pad = (-len(packed)) % 4
    if pad:
        packed = np.concatenate([packed, np.zeros(pad, dtype=np.uint8)])
    with open(path, "wb") as fh:
        fh.write(int(bits.size).to_bytes(8, "little"))
        fh.write(packed.tobytes())


def write_packed_bit_file(words, n: int, path: str) -> None:
    """Bit file from packed decoder words (bit t&31 of word t>>5) without unpacking:
    byte-identical to write_bit_file(unpacked bits)."""
    w = np.asarray(words).view(np.uint8).reshape(-1)
    nbytes = (n + 7) // 8
    body = np.array(w[:nbytes], dtype=np.uint8)
    if n % 8:
        body[-1] &= (1 << (n % 8)) - 1
    pad = (-nbytes) % 4
    with open(path, "wb") as fh:
        fh.write(int(n).to_bytes(8, "little"))
        fh.write(body.tobytes())
        fh.write(bytes(pad))


def read_bit_file(path: str) -> np.ndarray:
    """cli.read_bit_file (cli.py:42-52); ValueError on truncated files like the reference."""
    with open(path, "rb") as fh:
        raw = fh.read()
    if len(raw) < 8:
        raise ValueError(f"{path}: truncated bit file")
    n = int.from_bytes(raw[:8], "little")
    bits = np.unpackbits(np.frombuffer(raw[8:], dtype=np.uint8), bitorder="little")
    if bits.size < n:
        raise ValueError(f"{path}: bit file shorter than its header count")
    return bits[:n]


def write_llr_file(llr_flat, path: str, dtype: str) -> None:
    """cli.write_llr_file (cli.py:55-57): stage-major, polynomial-minor scalars."""
    np.asarray(llr_flat).astype(_llr_np_dtype(dtype)).tofile(path)


def read_llr_file(path: str, dtype: str) -> np.ndarray:
    """cli.read_llr_file (cli.py:60-62): float64 flat array."""
    return np.fromfile(path, dtype=_llr_np_dtype(dtype)).astype(np.float64)


def _to_int8(block: np.ndarray) -> np.ndarray:
    if block.size and (not np.all(np.isfinite(block)) or np.any(block != np.rint(block))):
        raise ValueError("LLR file holds non-integer values: the B200 decoder is exact on integer "
                         "(int8-quantised) LLRs; quantise with quantize_llr first")
    if block.size and (block.min() < -128 or block.max() > 127):
        raise ValueError("LLR values must lie in [-128, 127] (int8 quantised LLRs)")
    return block.astype(np.int8)


def decode_llr_file(llr_path: str, dtype: str, spec: CodeSpec, frame_len: int, overlap: int,
                    out_path: str | None = None, *, windows_per_piece: int = 1 << 18, stream=None) -> np.ndarray:
    """Decode an LLR file (the ``vitertile decode --llr-in F --frame-len F --overlap V``
    path, cli.py:135-173) with the B200 kernels, streaming it in pieces of
    ``windows_per_piece`` windows.  Returns the packed int32 words; writes the
    reference's decode output (raw little-endian packed bits) to ``out_path``
    when given."""
    torch = _torch()
    b = spec.outputs_per_bit
    npdt = np.dtype(_llr_np_dtype(dtype))
    total = os.path.getsize(llr_path) // npdt.itemsize
    if total % b:
        raise ValueError("LLR file length is not a multiple of the code rate denominator")
    n = total // b
    if n < 1:
        raise ValueError("LLR file is empty")
    if frame_len < 1 or overlap < 0:
        raise ValueError("frame length must be >= 1 and overlap >= 0")
    mm = np.memmap(llr_path, dtype=npdt, mode="r", shape=(n, b))
    code = _code(spec)
    nw = -(-n // frame_len)
    nwords = (n + 31) // 32
    dev = torch.device("cuda", torch.cuda.current_device())
    bits = torch.zeros(nwords, dtype=torch.int32, device=dev)
    per = max(1, int(windows_per_piece))
    max_stages = min(n, per * frame_len + 2 * overlap + 16)
    host = torch.empty(max_stages * b, dtype=torch.int8, pin_memory=True)
    llr_dev = torch.empty(((max_stages * b + 15) // 16) * 16, dtype=torch.int8, device=dev)
    s = stream or torch.cuda.current_stream(dev)
    for w0 in range(0, nw, per):
        w1 = min(nw, w0 + per)
        st0 = (max(0, w0 * frame_len - overlap) // 16) * 16  # the C ABI wants st0 % 16 == 0
        st1 = min(n, min(w1 * frame_len, n) + overlap)
        q = _to_int8(np.asarray(mm[st0:st1], dtype=np.float64)).reshape(-1)
        host[: q.size].copy_(torch.from_numpy(q))  # (the previous piece was synchronised below)
        with torch.cuda.stream(s):
            llr_dev[: q.size].copy_(host[: q.size], non_blocking=True)
        need = lib().vt_workspace_bytes(ctypes.byref(code), n, int(frame_len), int(overlap), w0, w1)
        ws = _workspace(need, s)
        check(lib().vt_decode_stream_range(ctypes.byref(code), _ptr(llr_dev), st0, st1, n, int(frame_len),
                                           int(overlap), w0, w1, _ptr(bits), None, _ptr(ws), ws.numel(),
                                           _stream_ptr(s)))
        s.synchronize()
    words = bits.cpu().numpy()
    if out_path is not None:
        if n % 8:
            raise ValueError("decoded bit count is not byte aligned; refusing to truncate")
        with open(out_path, "wb") as fh:
            fh.write(words.view(np.uint8)[: n // 8].tobytes())
    return words
