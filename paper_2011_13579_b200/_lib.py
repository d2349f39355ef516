"""ctypes binding of the in-tree sm_100a library (include/vitertile_b200.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is present, every decode call raises.
"""
from __future__ import annotations

import ctypes
import os

__all__ = ["VtCode", "lib", "check", "LIB_PATH", "VT_MAX_OUTPUTS"]

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libvitertile_b200.so")
VT_MAX_OUTPUTS = 8

VT_OK, VT_EINVAL, VT_EUNSUPPORTED, VT_EWORKSPACE, VT_ECUDA = 0, -1, -2, -3, -4


class VtCode(ctypes.Structure):
    _fields_ = [("K", ctypes.c_int32), ("B", ctypes.c_int32), ("gens", ctypes.c_uint32 * VT_MAX_OUTPUTS)]

    @classmethod
    def from_spec(cls, spec) -> "VtCode":
        c = cls()
        c.K = int(spec.constraint_length)
        c.B = len(spec.generators)
        if c.B > VT_MAX_OUTPUTS:
            raise ValueError(f"at most {VT_MAX_OUTPUTS} generator polynomials are supported")
        for i, g in enumerate(spec.generators):
            c.gens[i] = int(g)
        return c


_lib = None


def lib():
    """Load libvitertile_b200.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build the sm_100a extension first "
            "(python -c 'import __graft_entry__ as g; g.build()' or python paper_2011_13579_b200/build.py)")
    L = ctypes.CDLL(LIB_PATH)
    p, i64, vp = ctypes.POINTER, ctypes.c_int64, ctypes.c_void_p
    code_p = p(VtCode)
    L.vt_version.restype = ctypes.c_int
    L.vt_code_supported.argtypes = [code_p]
    L.vt_code_supported.restype = ctypes.c_int
    L.vt_last_error.restype = ctypes.c_char_p
    L.vt_load_code_module.argtypes = [ctypes.c_char_p]
    L.vt_load_code_module.restype = ctypes.c_int
    L.vt_workspace_bytes.argtypes = [code_p, i64, i64, i64, i64, i64]
    L.vt_workspace_bytes.restype = ctypes.c_size_t
    L.vt_decode_stream.argtypes = [code_p, vp, i64, i64, i64, vp, vp, vp, ctypes.c_size_t, vp]
    L.vt_decode_stream_range.argtypes = [code_p, vp, i64, i64, i64, i64, i64, i64, i64, vp, vp, vp,
                                         ctypes.c_size_t, vp]
    L.vt_decode_frames.argtypes = [code_p, vp, i64, i64, vp, vp, vp, ctypes.c_size_t, vp]
    L.vt_decode_stream_host.argtypes = [code_p, vp, i64, i64, i64, vp, vp, vp, vp, ctypes.c_size_t,
                                        ctypes.c_int, vp]
    L.vt_workspace_bytes_host.argtypes = [code_p, i64, i64, i64, i64, i64, ctypes.c_int]
    L.vt_workspace_bytes_host.restype = ctypes.c_size_t
    L.vt_shard_range.argtypes = [i64, i64, i64, ctypes.c_int, ctypes.c_int, p(i64)]
    L.vt_decode_stream_host_multi.argtypes = [code_p, vp, i64, i64, i64, vp, ctypes.c_int, p(ctypes.c_int), p(vp),
                                              p(vp), p(vp), p(ctypes.c_size_t), ctypes.c_int]
    L.vt_matrix_forward.argtypes = [code_p, vp, i64, i64, vp, vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, vp,
                                    vp, vp, vp, vp]
    L.vt_matrix_forward.restype = ctypes.c_int
    L.vt_channel_awgn.argtypes = [code_p, ctypes.c_uint64, ctypes.c_uint32, i64, i64, ctypes.c_float, ctypes.c_float,
                                  ctypes.c_int, vp, vp, vp]
    L.vt_count_bit_errors.argtypes = [vp, vp, i64, vp, vp]
    L.vt_workspace_bytes_r4perm.argtypes = [code_p, i64, i64, i64, i64, i64]
    L.vt_workspace_bytes_r4perm.restype = ctypes.c_size_t
    L.vt_decode_stream_r4perm.argtypes = [code_p, vp, vp, i64, i64, i64, i64, i64, i64, i64, vp, vp, vp,
                                          ctypes.c_size_t, vp]
    L.vt_forward_batch.argtypes = [code_p, vp, i64, i64, vp, ctypes.c_int, ctypes.c_int, vp, vp, vp, vp]
    L.vt_pack_llr_f64.argtypes = [vp, i64, i64, i64, vp, ctypes.c_int]
    L.vt_pack_llr_f64.restype = ctypes.c_int
    L.vt_traceback_batch.argtypes = [code_p, vp, vp, i64, i64, vp, vp]
    for fn in ("vt_shard_range", "vt_decode_stream_host_multi", "vt_decode_stream", "vt_decode_stream_range", "vt_decode_frames", "vt_decode_stream_host",
               "vt_channel_awgn", "vt_count_bit_errors", "vt_decode_stream_r4perm", "vt_forward_batch",
               "vt_traceback_batch"):
        getattr(L, fn).restype = ctypes.c_int
    _lib = L
    return L


def check(rc: int) -> None:
    """Map a C-ABI status to the reference's error convention (ValueError)."""
    if rc == VT_OK:
        return
    msg = lib().vt_last_error().decode(errors="replace")
    if rc == VT_EINVAL:
        raise ValueError(msg)
    if rc == VT_EUNSUPPORTED:
        raise NotImplementedError(msg)
    raise RuntimeError(f"vitertile_b200 error {rc}: {msg}")
