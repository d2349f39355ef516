"""Convolutional-code description and host-side trellis tables.

Mirrors the public surface of the reference's ``vitertile.codes`` that the
decode path consumes (pkg/src/vitertile/codes.py:51-107 CodeSpec,
183-193 branch_output, 205-230 encode/encode_batch, 351-412 BOMAT/dragonfly
groups, 477-480 default_spec).  Only table generation lives here; decoding
runs in the sm_100a kernels.

State convention (codes.py:1-6): a state is the previous K-1 input bits with
the newest bit in the MSB; input u moves state i to (u << (K-2)) | (i >> 1);
output bit b is the parity of g_b AND ((u << (K-1)) | i).
"""
from __future__ import annotations

import sys
from dataclasses import dataclass
from functools import lru_cache
from typing import Sequence

import numpy as np

if sys.version_info >= (3, 11):
    import tomllib as _toml
else:  # pragma: no cover
    import tomli as _toml

__all__ = [
    "CodeSpec",
    "DragonflyGroup",
    "default_spec",
    "branch_output",
    "encode",
    "encode_batch",
    "compute_bomat",
    "identical_bomat_classes",
    "find_dragonfly_groups",
]


def _par(x: int) -> int:
    return int(x).bit_count() & 1


@dataclass(frozen=True)
class CodeSpec:
    """Feed-forward convolutional code: constraint length + generator polynomials
    (codes.py:51-107; same validation and derived sizes)."""

    constraint_length: int
    generators: tuple[int, ...]

    def __post_init__(self) -> None:
        k = int(self.constraint_length)
        if k < 3:
            raise ValueError(f"constraint length must be >= 3, got {k}")
        gens = tuple(int(g) for g in self.generators)
        if len(gens) < 2:
            raise ValueError("need at least 2 generator polynomials")
        bad = [g for g in gens if g < 0 or g >= (1 << k)]
        if bad:
            raise ValueError(f"generator {bad[0]:#o} does not fit in {k} bits")
        object.__setattr__(self, "constraint_length", k)
        object.__setattr__(self, "generators", gens)

    @property
    def outputs_per_bit(self) -> int:
        return len(self.generators)

    @property
    def num_states(self) -> int:
        return 1 << (self.constraint_length - 1)

    @property
    def num_butterflies(self) -> int:
        return 1 << (self.constraint_length - 2)

    def check_radix_log(self, rho: int) -> None:
        if rho < 1 or rho > self.constraint_length - 1:
            raise ValueError(f"stage width {rho} out of range for K={self.constraint_length}")

    def num_dragonflies(self, rho: int) -> int:
        self.check_radix_log(rho)
        return 1 << (self.constraint_length - 1 - rho)

    @property
    def octal_generators(self) -> tuple[str, ...]:
        return tuple(f"{g:o}" for g in self.generators)

    @classmethod
    def from_octal(cls, constraint_length: int, polynomials: Sequence[int | str]) -> "CodeSpec":
        return cls(int(constraint_length), tuple(int(str(p), 8) for p in polynomials))

    @classmethod
    def from_config(cls, path: str) -> "CodeSpec":
        with open(path, "rb") as fh:
            cfg = _toml.load(fh)
        return cls.from_octal(int(cfg["k"]), cfg["polynomials"])


@lru_cache(maxsize=None)
def default_spec() -> CodeSpec:
    """K=7 rate-1/2 (171, 133) (codes.py:477-480)."""
    return CodeSpec(7, (0o171, 0o133))


def branch_output(state: int, input_bit: int, spec: CodeSpec) -> tuple[int, tuple[int, ...]]:
    """One trellis branch: (next state, output bits) (codes.py:183-193)."""
    k = spec.constraint_length
    if state < 0 or state >= spec.num_states:
        raise ValueError(f"state {state} out of range")
    if input_bit not in (0, 1):
        raise ValueError("input bit must be 0 or 1")
    reg = (input_bit << (k - 1)) | state
    return (input_bit << (k - 2)) | (state >> 1), tuple(_par(g & reg) for g in spec.generators)


def encode_batch(bits2d: np.ndarray, spec: CodeSpec) -> np.ndarray:
    """Encode frames (F, N) from the zero state -> coded bits (F, N, B) (codes.py:216-230).

    Vectorised as a GF(2) convolution: output b at stage t is the XOR of the
    inputs t-d for every tap d of generator b (tap d=0 is bit K-1)."""
    bits2d = np.asarray(bits2d, dtype=np.uint8)
    f, n = bits2d.shape
    k = spec.constraint_length
    hist = np.zeros((f, n + k - 1), dtype=np.uint8)
    hist[:, k - 1:] = bits2d & 1
    out = np.empty((f, n, spec.outputs_per_bit), dtype=np.uint8)
    for b, g in enumerate(spec.generators):
        acc = np.zeros((f, n), dtype=np.uint8)
        for d in range(k):
            if (g >> (k - 1 - d)) & 1:
                acc ^= hist[:, k - 1 - d: k - 1 - d + n]
        out[:, :, b] = acc
    return out


def encode(bits, spec: CodeSpec) -> np.ndarray:
    """Stage-major, polynomial-minor coded stream of length N*B (codes.py:205-213)."""
    arr = np.asarray(bits, dtype=np.uint8)
    if arr.ndim != 1 or arr.size == 0:
        raise ValueError("input must be a non-empty 1-D bit sequence")
    if np.any(arr > 1):
        raise ValueError("input must contain only bits")
    return encode_batch(arr[None, :], spec)[0].reshape(-1)


# ---------------------------------------------------------------------------
# branch-output matrices (paper's A operand) and dragonfly groups, used for the
# tile-op counters of decode_matrix_batch (matrix.py:129-265)
# ---------------------------------------------------------------------------


def _dragonfly_state(f: int, y: int, x: int, rho: int, k: int) -> int:
    # codes.py:276-288: pre-bubble bits of y above, dragonfly index, post-bubble bits
    pre = (y % (1 << rho)) >> (rho - x)
    post = y % (1 << (rho - x))
    return (pre << (k - x - 1)) + (f << (rho - x)) + post


def compute_bomat(f: int, rho: int, spec: CodeSpec) -> np.ndarray:
    """+-1 super-branch output matrix of dragonfly f, rows (right j, left i) ->
    row j*2^rho + i (codes.py:351-365)."""
    n = 1 << rho
    k = spec.constraint_length
    rows = np.empty((n * n, rho * spec.outputs_per_bit), dtype=np.int8)
    for j in range(n):
        for i in range(n):
            st = _dragonfly_state(f, i, 0, rho, k)
            col = []
            for x in range(rho):  # input bits along the unique path, earliest first
                st, bo = branch_output(st, (j >> x) & 1, spec)
                col.extend(1 - 2 * v for v in bo)
            rows[j * n + i] = col
    return rows


def identical_bomat_classes(rho: int, spec: CodeSpec) -> list[tuple[int, ...]]:
    """Dragonflies grouped by identical output matrix (codes.py:374-380)."""
    seen: dict[bytes, list[int]] = {}
    for f in range(spec.num_dragonflies(rho)):
        seen.setdefault(compute_bomat(f, rho, spec).tobytes(), []).append(f)
    return [tuple(v) for v in seen.values()]


@dataclass(frozen=True)
class DragonflyGroup:
    representative: int
    members: tuple[int, ...]
    permutations: dict[int, tuple[int, ...]]


def find_dragonfly_groups(rho: int, spec: CodeSpec) -> list[DragonflyGroup]:
    """Maximal groups whose output matrices are left-state permutations of each
    other (codes.py:383-412): equal multisets of left-state signatures."""
    n = 1 << rho
    sig = {}
    by_key: dict[tuple, list[int]] = {}
    for f in range(spec.num_dragonflies(rho)):
        m = compute_bomat(f, rho, spec)
        s = [tuple(tuple(int(v) for v in m[j * n + i]) for j in range(n)) for i in range(n)]
        sig[f] = s
        by_key.setdefault(tuple(sorted(s)), []).append(f)
    groups = []
    for members in by_key.values():
        rep = min(members)
        perms = {}
        for f in members:
            free = list(range(n))
            perm = []
            for want in sig[rep]:
                pos = next(p for p in free if sig[f][p] == want)
                free.remove(pos)
                perm.append(pos)
            perms[f] = tuple(perm)
        groups.append(DragonflyGroup(rep, tuple(sorted(members)), perms))
    return sorted(groups, key=lambda g: g.representative)
