"""Throughput of the tensor-core tile decoder (decode_matrix_batch's kernel,
csrc/vt_tiles.cu) vs the fused ACS kernel on the same frames: K=7 r1/2 frames of
256 stages, device-resident, CUDA events."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2011_13579_b200 as vt  # noqa: E402
from paper_2011_13579_b200.decoder import _matrix_frames_device  # noqa: E402

spec = vt.default_spec()
f, n = 1 << 16, 256
dev = torch.randint(-128, 128, (f, n, 2), dtype=torch.int8, device="cuda")
for name, cfg in (("radix2", vt.DecoderConfig(radix=2)), ("radix4-opt", vt.DecoderConfig(radix=4, optimized=True)),
                  ("radix2-half", vt.DecoderConfig(policy=vt.PrecisionPolicy(accumulator="half")))):
    _matrix_frames_device(dev, spec, cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        _, _, ops = _matrix_frames_device(dev, spec, cfg)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 3
    tiles = ops * f  # 16x16x16 tile ops per launch
    print(f"tile decoder {name}: {f * n / ms / 1e6:.3f} Gbps  {ms:.2f} ms  {tiles / ms / 1e6:.3f} G tile-ops/s "
          f"({tiles * 2 * 4096 / ms / 1e9:.4f} TFLOP/s dense-equivalent)", flush=True)
words = torch.zeros((f * n + 31) // 32, dtype=torch.int32, device="cuda")
flat = dev.reshape(f * n, 2)
vt.decode_stream_device(flat, spec, n, 0, out=words)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    vt.decode_stream_device(flat, spec, n, 0, out=words)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"fused 16x2 ACS kernel, same frames: {f * n / ms / 1e6:.3f} Gbps  {ms:.3f} ms")
