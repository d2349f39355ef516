"""The paper's tile packings (matrix.py:129-265 of the reference) as tensor-core
fragment programs for ``vt_matrix_forward`` (csrc/vt_tiles.cu).

A tile is one 16x16x16 op D = A x B + C of the paper's formulation
(tile.py:61-89):

* radix 2 (pack_radix2, matrix.py:129-180): 4x4 diagonal blocks, one per group of
  <= 4 butterflies sharing a branch-output matrix; column = butterfly beta,
  rows (i0 j0, i1 j0, i0 j1, i1 j1); B holds the stage's LLRs, C the left-state
  metrics; output state beta + lj * S/2 picks row 2 lj + 1 over 2 lj on ties;
* radix 4 (pack_radix4, matrix.py:187-265): 16 x 2B horizontal blocks, one per
  group of <= 4 dragonflies (identical matrices, or with optimized=True the
  dragonfly-permutation groups of find_dragonfly_groups, whose members' metrics
  enter C in the representative's left-state order); output state
  j * S/4 + f picks the last maximal of its 4 candidate rows and records
  perm[k].

``program()`` turns a packing into the per-lane fragment tables of
mma.sync.m16n8k16 (A row-major 16x16 f16, B col-major 16x8 f16 twice, C/D
16x8 f32 twice): lane = 4 g + q holds A rows g, g+8 x cols 2q.., 2q+8..;
B rows 2q.., 2q+8.. x col g (+8 for the second n-block); C/D rows g, g+8 x
cols 2q, 2q+1 (+8).
"""
from __future__ import annotations

import ctypes
import threading
from dataclasses import dataclass

import numpy as np

from .codes import CodeSpec, compute_bomat, find_dragonfly_groups, identical_bomat_classes

TILE, BLOCK = 16, 4

__all__ = ["TileSet", "radix2_tiles", "radix4_tiles", "VtTileProgram", "device_program"]


@dataclass
class TileSet:
    """One packing: per tile the A matrix, the B placements (row, col, llr index),
    the C gathers (row, col) -> state, and the outputs (candidate (row, col) list,
    state, survivor code per candidate)."""

    ncand: int
    nllr: int
    a: list                 # (16, 16) float arrays
    b_place: list           # [{(row, col): llr index}]
    c_gather: list          # [{(row, col): state}]
    outputs: list           # [[(cands [(row, col)], state, codes)]]
    effective: bool = True  # radix-4 optimisation in effect (matrix.py:206-220)

    @property
    def ntiles(self) -> int:
        return len(self.a)


def _tile_chunks(blocks):
    return [blocks[i:i + TILE // BLOCK] for i in range(0, len(blocks), TILE // BLOCK)]


def radix2_tiles(spec: CodeSpec) -> TileSet:
    """pack_radix2 (matrix.py:129-180)."""
    b = spec.outputs_per_bit
    if b > BLOCK:
        raise ValueError(f"butterfly output matrix width {b} exceeds block width {BLOCK}")
    half = spec.num_butterflies
    blocks = []
    for cls in identical_bomat_classes(1, spec):
        m = compute_bomat(cls[0], 1, spec)
        blocks += [(m, list(cls[i:i + BLOCK])) for i in range(0, len(cls), BLOCK)]
    ts = TileSet(2, b, [], [], [], [])
    for tile in _tile_chunks(blocks):
        a = np.zeros((TILE, TILE), dtype=np.float32)
        bp, cg, outs = {}, {}, []
        for d, (m, betas) in enumerate(tile):
            base = BLOCK * d
            a[base:base + 4, base:base + b] = m
            for slot, beta in enumerate(betas):
                col = base + slot
                for bb in range(b):
                    bp[(base + bb, col)] = bb
                for r, left in enumerate((2 * beta, 2 * beta + 1, 2 * beta, 2 * beta + 1)):
                    cg[(base + r, col)] = left
                for lj in range(2):
                    outs.append(([(base + 2 * lj, col), (base + 2 * lj + 1, col)], beta + lj * half, (0, 1)))
        ts.a.append(a)
        ts.b_place.append(bp)
        ts.c_gather.append(cg)
        ts.outputs.append(outs)
    return ts


def radix4_tiles(spec: CodeSpec, optimized: bool = False) -> TileSet:
    """pack_radix4 (matrix.py:187-265), incl. the fall-back when the dragonfly groups
    need no fewer blocks than the identical-matrix classes."""
    b = spec.outputs_per_bit
    if 2 * b > BLOCK:
        raise ValueError(f"super-branch output width {2 * b} exceeds block width {BLOCK}")
    ident = (0, 1, 2, 3)
    plain = []
    for cls in identical_bomat_classes(2, spec):
        m = compute_bomat(cls[0], 2, spec)
        plain += [(m, [(f, ident) for f in cls[i:i + BLOCK]]) for i in range(0, len(cls), BLOCK)]
    blocks, effective = plain, False
    if optimized:
        grouped = []
        for grp in find_dragonfly_groups(2, spec):
            m = compute_bomat(grp.representative, 2, spec)
            mem = [(f, grp.permutations[f]) for f in grp.members]
            grouped += [(m, mem[i:i + BLOCK]) for i in range(0, len(mem), BLOCK)]
        if len(grouped) < len(plain):
            blocks, effective = grouped, True
    step = spec.num_dragonflies(2)
    ts = TileSet(4, 2 * b, [], [], [], [], effective)
    for tile in _tile_chunks(blocks):
        a = np.zeros((TILE, TILE), dtype=np.float32)
        bp, cg, outs = {}, {}, []
        for d, (m, members) in enumerate(tile):
            base = BLOCK * d
            a[:, base:base + 2 * b] = m
            for slot, (f, perm) in enumerate(members):
                col = base + slot
                for bb in range(2 * b):
                    bp[(base + bb, col)] = bb
                for j in range(4):
                    for i in range(4):
                        cg[(4 * j + i, col)] = 4 * f + perm[i]
                    outs.append(([(4 * j + i, col) for i in range(4)], j * step + f, tuple(perm)))
        ts.a.append(a)
        ts.b_place.append(bp)
        ts.c_gather.append(cg)
        ts.outputs.append(outs)
    return ts


def _h16(x: float) -> int:
    return int(np.array(x, dtype=np.float16).view(np.uint16))


def fragment_tables(ts: TileSet) -> dict:
    """Per-lane mma.sync.m16n8k16 fragment tables of a tile set (layout in the module
    docstring); arrays ready for the device."""
    nt = ts.ntiles
    nout = max(len(o) for o in ts.outputs)
    a_frag = np.zeros((nt, 32, 4), dtype=np.uint32)
    b_sel = np.full((nt, 32, 8), -1, dtype=np.int8)
    c_state = np.full((nt, 32, 8), -1, dtype=np.int16)
    cand = np.zeros((nt, nout, 4), dtype=np.uint8)
    out_state = np.full((nt, nout), -1, dtype=np.int16)
    code = np.zeros((nt, nout, 4), dtype=np.uint8)
    for t in range(nt):
        a = ts.a[t]
        for lane in range(32):
            g, q = lane >> 2, lane & 3
            pairs = ((g, 2 * q), (g + 8, 2 * q), (g, 2 * q + 8), (g + 8, 2 * q + 8))
            for r, (row, col) in enumerate(pairs):
                a_frag[t, lane, r] = _h16(a[row, col]) | (_h16(a[row, col + 1]) << 16)
            for nb in range(2):
                bcol = nb * 8 + g
                for i, row in enumerate((2 * q, 2 * q + 1, 2 * q + 8, 2 * q + 9)):
                    b_sel[t, lane, nb * 4 + i] = ts.b_place[t].get((row, bcol), -1)
                c0 = nb * 8 + 2 * q
                for i, (row, col) in enumerate(((g, c0), (g, c0 + 1), (g + 8, c0), (g + 8, c0 + 1))):
                    c_state[t, lane, nb * 4 + i] = ts.c_gather[t].get((row, col), -1)
        for o, (cands, state, codes) in enumerate(ts.outputs[t]):
            for k, (row, col) in enumerate(cands):
                cand[t, o, k] = row * 16 + col
                code[t, o, k] = codes[k]
            out_state[t, o] = state
    return {"ntiles": nt, "nout": nout, "ncand": ts.ncand, "nllr": ts.nllr, "a_frag": a_frag, "b_sel": b_sel,
            "c_state": c_state, "cand": cand, "out_state": out_state, "code": code}


class VtTileProgram(ctypes.Structure):
    _fields_ = [("ntiles", ctypes.c_int32), ("nout", ctypes.c_int32), ("ncand", ctypes.c_int32),
                ("nllr", ctypes.c_int32), ("a_frag", ctypes.c_void_p), ("b_sel", ctypes.c_void_p),
                ("c_state", ctypes.c_void_p), ("cand", ctypes.c_void_p), ("out_state", ctypes.c_void_p),
                ("code", ctypes.c_void_p)]


_cache: dict = {}
_cache_lock = threading.Lock()


def device_program(spec: CodeSpec, radix: int, optimized: bool = False):
    """(VtTileProgram with device tables, TileSet) for the code and radix on the current
    device; cached (the tensors stay alive in the cache)."""
    import torch
    key = (int(spec.constraint_length), tuple(int(g) for g in spec.generators), radix, bool(optimized),
           torch.cuda.current_device())
    with _cache_lock:
        hit = _cache.get(key)
        if hit is not None:
            return hit[0], hit[1]
        ts = radix2_tiles(spec) if radix == 2 else radix4_tiles(spec, optimized)
        tab = fragment_tables(ts)
        dev = {k: torch.from_numpy(np.ascontiguousarray(v.view(np.int32) if v.dtype == np.uint32 else v)).cuda()
               for k, v in tab.items() if isinstance(v, np.ndarray)}
        prog = VtTileProgram(tab["ntiles"], tab["nout"], tab["ncand"], tab["nllr"],
                             *[dev[k].data_ptr() for k in ("a_frag", "b_sel", "c_state", "cand", "out_state", "code")])
        _cache[key] = (prog, ts, dev)
        return prog, ts
