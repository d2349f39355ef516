"""Decode throughput of one code through each kernel form (device-resident
stream, CUDA events), for A/B runs of kernel variants:
  python tools/code_bench.py k7r3 --log2n 28 --variants 16x2,s32 [--so a.so,b.so]
Prints one line per (library, variant): Gbps, ms per decode."""
import argparse
import os
import shutil
import subprocess
import sys

CODES = {"k7r2": (7, (0o171, 0o133)), "k7r3": (7, (0o133, 0o171, 0o165)), "k9r2": (9, (0o753, 0o561)),
         "k8r2": (8, (0o247, 0o371)), "k5r2": (5, (0o23, 0o35))}


def one(code, log2n, f, v, variant, steps):
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    if variant:
        os.environ["VT_KERNEL_VARIANT"] = variant
    import paper_2011_13579_b200 as vt
    from bench import make_stream
    k, gens = CODES[code]
    dev = torch.device("cuda", 0)
    n = 1 << log2n
    _, q = make_stream(torch, n, seed=77, device=dev, gens=gens, k=k)
    o = torch.zeros((n + 31) // 32, dtype=torch.int32, device=dev)
    spec = vt.CodeSpec(k, gens)
    s = torch.cuda.current_stream()
    for _ in range(3):
        vt.decode_stream_device(q, spec, f, v, out=o, stream=s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(s)
    for _ in range(steps):
        vt.decode_stream_device(q, spec, f, v, out=o, stream=s)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    print(f"{code} n=2^{log2n} F={f} V={v} variant={variant or 'default'}: {n / (ms * 1e-3) / 1e9:.2f} Gbps "
          f"({ms:.3f} ms)", flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("code", choices=sorted(CODES))
    ap.add_argument("--log2n", type=int, default=28)
    ap.add_argument("--frame", type=int, default=256)
    ap.add_argument("--overlap", type=int, default=42)
    ap.add_argument("--variants", default="")
    ap.add_argument("--so", default="", help="comma-separated libraries swapped in turn (each run in a subprocess)")
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--one", action="store_true", help=argparse.SUPPRESS)
    a = ap.parse_args()
    variants = a.variants.split(",") if a.variants else [""]
    if a.one:
        one(a.code, a.log2n, a.frame, a.overlap, variants[0], a.steps)
        return
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "paper_2011_13579_b200", "libvitertile_b200.so")
    libs = a.so.split(",") if a.so else [""]
    keep = lib + ".orig"
    if a.so:
        shutil.copy(lib, keep)
    try:
        for rep in range(2):
            for so in libs:
                if so:
                    shutil.copy(so, lib)
                for var in variants:
                    print(f"[{os.path.basename(so) or 'in-tree'} rep {rep}] ", end="", flush=True)
                    subprocess.run([sys.executable, __file__, a.code, "--one", "--log2n", str(a.log2n), "--frame",
                                    str(a.frame), "--overlap", str(a.overlap), "--variants", var, "--steps",
                                    str(a.steps)], check=False)
    finally:
        if a.so:
            shutil.move(keep, lib)


if __name__ == "__main__":
    main()
