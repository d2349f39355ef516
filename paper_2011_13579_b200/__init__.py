"""vitertile-B200: framed soft-decision Viterbi decoding on sm_100a.

Drop-in for the decode/encode API of the reference ``vitertile`` package
(pkg/src/vitertile/__init__.py:5-20 plus framing/reference/channel entry
points).  Decoding runs in hand-written sm_100a kernels behind the C ABI of
include/vitertile_b200.h; the Python layer only validates, moves buffers and
unpacks bits.
"""
from .codes import (
    CodeSpec,
    DragonflyGroup,
    branch_output,
    compute_bomat,
    default_spec,
    encode,
    encode_batch,
    find_dragonfly_groups,
    identical_bomat_classes,
)
from .decoder import (
    DecoderConfig,
    MatrixDecodeResult,
    PrecisionPolicy,
    SoftFrame,
    TileOpCounter,
    decode_batch,
    decode_matrix,
    decode_matrix_batch,
    decode_reference,
    decode_stream,
    decode_stream_device,
    decode_stream_host,
    quantize_llr,
    workspace_bytes,
    release_workspaces,
)
from . import fileio  # noqa: F401  (cli.py file formats)
from . import sharding  # noqa: F401  (multi-GPU window shards)
from .framing import DEFAULT_FRAME_LEN, DEFAULT_OVERLAP, FramePlan, Window, plan_frames

__all__ = [
    "CodeSpec",
    "DecoderConfig",
    "PrecisionPolicy",
    "SoftFrame",
    "TileOpCounter",
    "MatrixDecodeResult",
    "DragonflyGroup",
    "Window",
    "FramePlan",
    "DEFAULT_FRAME_LEN",
    "DEFAULT_OVERLAP",
    "plan_frames",
    "decode_stream",
    "decode_stream_device",
    "decode_stream_host",
    "decode_batch",
    "decode_reference",
    "decode_matrix",
    "decode_matrix_batch",
    "default_spec",
    "encode",
    "encode_batch",
    "branch_output",
    "compute_bomat",
    "identical_bomat_classes",
    "find_dragonfly_groups",
    "quantize_llr",
    "workspace_bytes",
    "release_workspaces",
]

__version__ = "0.1.0"
