"""Frame sharding across GPUs.

Windows of ``plan_frames(N, F, V)`` are independent (framing.py:96-141:
"Windows are independent; results do not depend on execution order"), so a
stream shards over G ranks with no data exchange: rank g decodes the
contiguous window range [w0, w1) from the stage range [st0, st1) (its emit
ranges plus a V-stage halo each side) and writes a disjoint range of packed
output words.  The only collective is an optional all_gather of the packed
bits (``gather_bits``).  ``shard_windows`` is the Python mirror of the C ABI's
``vt_shard_range`` (the split ``vt_decode_stream_host_multi`` uses).
"""
from __future__ import annotations

from dataclasses import dataclass

__all__ = ["Shard", "shard_windows", "decode_stream_sharded", "gather_bits"]


@dataclass(frozen=True)
class Shard:
    rank: int
    w0: int  # first window (inclusive)
    w1: int  # last window (exclusive)
    st0: int  # first stage held by the rank's LLR buffer (multiple of 16)
    st1: int  # one past the last stage held
    word0: int  # first packed output word the rank completes
    word1: int  # one past the last packed output word the rank completes

    @property
    def num_windows(self) -> int:
        return self.w1 - self.w0


def shard_windows(n: int, frame_len: int, overlap: int, world: int, rank: int) -> Shard:
    """Contiguous, balanced window range of ``rank`` and the stage halo it needs."""
    if n < 1 or frame_len < 1 or overlap < 0:
        raise ValueError("bad stream geometry")
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    nw = -(-n // frame_len)
    w0, w1 = nw * rank // world, nw * (rank + 1) // world
    st0 = (max(0, w0 * frame_len - overlap) // 16) * 16
    st1 = min(n, min(w1 * frame_len, n) + overlap) if w1 > w0 else st0
    # words whose every bit is emitted by this rank's windows (boundary words may be shared)
    e0, e1 = w0 * frame_len, min(w1 * frame_len, n)
    word0 = -(-e0 // 32)
    word1 = (n + 31) // 32 if w1 == nw else e1 // 32
    return Shard(rank, w0, w1, st0, st1, word0, max(word0, word1))


def decode_stream_sharded(llr_shard_nb, spec, n: int, frame_len: int, overlap: int, shard: Shard, out=None,
                          stream=None):
    """Decode this rank's windows from its int8 (st1-st0, B) device buffer.

    Returns the packed int32 word tensor of the whole stream with this rank's
    words filled (other words zero)."""
    import ctypes

    import torch

    from ._lib import check, lib
    from .decoder import _code, _ptr, _stream_ptr, _workspace

    code = _code(spec)
    llr_shard_nb = llr_shard_nb.contiguous()
    if llr_shard_nb.data_ptr() % 16:  # the kernels stage 16-byte words
        llr_shard_nb = llr_shard_nb.clone()
    nwords = (n + 31) // 32
    if out is None:
        out = torch.zeros(nwords, dtype=torch.int32, device=llr_shard_nb.device)
    if shard.num_windows == 0:
        return out
    need = lib().vt_workspace_bytes(ctypes.byref(code), n, frame_len, overlap, shard.w0, shard.w1)
    ws = _workspace(need, stream)
    check(lib().vt_decode_stream_range(ctypes.byref(code), _ptr(llr_shard_nb), shard.st0, shard.st1, n, frame_len,
                                       overlap, shard.w0, shard.w1, _ptr(out), None, _ptr(ws), ws.numel(),
                                       _stream_ptr(stream)))
    return out


def _edges(n: int, frame_len: int, sh: Shard) -> tuple[int, int]:
    """Words this shard shares with its neighbours (-1: none)."""
    if sh.num_windows == 0:
        return -1, -1
    e0, e1 = sh.w0 * frame_len, min(sh.w1 * frame_len, n)
    return (e0 // 32 if e0 % 32 else -1), (e1 // 32 if (e1 < n and e1 % 32) else -1)


def gather_bits(words, n: int, frame_len: int, overlap: int, group=None):
    """Assemble the whole stream's packed words on every rank from each rank's
    decode (``decode_stream_sharded``).  One ``all_gather`` of equal-size
    buffers -- each rank's own word range [word0, word1) padded to the longest,
    plus the <= 2 words it shares with its neighbours -- so only the words a rank
    wrote travel (NCCL and gloo both support it; NCCL has no bitwise
    reductions).  Shared words hold disjoint bits of two ranks and are OR-merged.
    Returns ``words`` with every word filled."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    shards = [shard_windows(n, frame_len, overlap, world, r) for r in range(world)]
    width = max(s.word1 - s.word0 for s in shards) + 2
    sh = shards[rank]
    buf = torch.zeros(width, dtype=words.dtype, device=words.device)
    own = sh.word1 - sh.word0
    buf[:own] = words[sh.word0:sh.word1]
    for k, idx in enumerate(_edges(n, frame_len, sh)):
        if idx >= 0:
            buf[width - 2 + k] = words[idx]
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    edge_words = []
    for r, s in enumerate(shards):
        words[s.word0:s.word1] = parts[r][:s.word1 - s.word0]
        for k, idx in enumerate(_edges(n, frame_len, s)):
            if idx >= 0:
                edge_words.append((idx, parts[r][width - 2 + k]))
    for idx, _ in edge_words:
        words[idx] = 0
    for idx, val in edge_words:
        words[idx] |= val
    return words
