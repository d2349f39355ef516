"""``python -m paper_2011_13579_b200``: the decode/encode commands of the reference
CLI (pkg/src/vitertile/cli.py:115-173) on the B200 decoder.

  encode  INFILE --out BITFILE                     (cli.py:115-124)
  decode  INFILE|--llr-in F --out OUT [--frame-len F --overlap V]   (cli.py:127-173)

Same file formats and arguments (--k, --poly, --llr-dtype, --frame-len,
--overlap, --radix, --optimized); decoding always runs the sm_100a kernels.
The scalar-reference path (no --radix) streams the LLR file through the
window-range kernel; --radix selects the tile-decoder semantics (radix-4
--optimized has its own tie order, matrix.py:329-333) on the whole file.
Without --frame-len the whole stream is one window, as the reference's
decode_batch / decode_matrix on a single frame.
"""
from __future__ import annotations

import argparse
import json
import sys

import numpy as np

from .codes import CodeSpec, encode
from .fileio import decode_llr_file, read_bit_file, write_bit_file, write_llr_file


def _spec(args) -> CodeSpec:
    polys = [p.strip() for p in str(args.poly).split(",") if p.strip()]
    spec = CodeSpec.from_octal(args.k, polys)
    if args.rate_den is not None and args.rate_den != spec.outputs_per_bit:
        raise SystemExit(f"--rate-den {args.rate_den} does not match {len(polys)} polynomials")
    return spec


def _cmd_encode(args) -> int:
    spec = _spec(args)
    with open(args.infile, "rb") as fh:
        data = fh.read()
    if not data:
        raise SystemExit("input file is empty")
    bits = np.unpackbits(np.frombuffer(data, dtype=np.uint8), bitorder="little")
    write_bit_file(encode(bits, spec), args.out)
    return 0


def _cmd_decode(args) -> int:
    import tempfile
    import os
    spec = _spec(args)
    b = spec.outputs_per_bit
    tmp = None
    if args.llr_in:
        path, dtype = args.llr_in, args.llr_dtype
    else:  # hard-decision bit file -> +-1 LLRs (cli.py:141-145)
        coded = read_bit_file(args.infile)
        if coded.size % b:
            raise SystemExit("coded bit count is not a multiple of the code rate denominator")
        fd, tmp = tempfile.mkstemp(suffix=".llr")
        os.close(fd)
        write_llr_file(1.0 - 2.0 * coded.astype(np.float64), tmp, "single")
        path, dtype = tmp, "single"
    try:
        n = (os.path.getsize(path) // (2 if dtype == "half" else 4)) // b
        f = args.frame_len or n
        v = args.overlap if args.frame_len else 0
        try:
            if args.radix is None:
                decode_llr_file(path, dtype, spec, f, v, args.out)
            else:
                from .decoder import DecoderConfig, decode_matrix, decode_stream
                from .fileio import read_llr_file
                from .framing import plan_frames
                llr = read_llr_file(path, dtype).reshape(-1, b).T
                cfg = DecoderConfig(radix=args.radix, optimized=args.optimized)
                if args.frame_len:
                    bits = decode_stream(llr, spec, plan_frames(n, f, v), decoder="matrix", config=cfg)
                else:
                    bits = decode_matrix(llr, spec, cfg).bits
                if bits.size % 8:
                    raise ValueError("decoded bit count is not byte aligned; refusing to truncate")
                with open(args.out, "wb") as fh:
                    fh.write(np.packbits(bits, bitorder="little").tobytes())
        except ValueError as exc:
            raise SystemExit(str(exc)) from None
    finally:
        if tmp:
            os.unlink(tmp)
    if args.stats:
        with open(args.stats, "w") as fh:
            json.dump({"decoder": "b200", "stages": n, "windows": -(-n // f)}, fh, indent=2)
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2011_13579_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    for name in ("encode", "decode"):
        p = sub.add_parser(name)
        p.add_argument("infile", nargs="?" if name == "decode" else None)
        p.add_argument("--out", required=True)
        p.add_argument("--k", type=int, default=7)
        p.add_argument("--poly", default="171,133")
        p.add_argument("--rate-den", type=int, default=None)
        if name == "decode":
            p.add_argument("--llr-in", default=None)
            p.add_argument("--llr-dtype", choices=("half", "single"), default="single")
            p.add_argument("--frame-len", type=int, default=0)
            p.add_argument("--overlap", type=int, default=64)
            p.add_argument("--radix", type=int, choices=(2, 4), default=None)
            p.add_argument("--optimized", action="store_true")
            p.add_argument("--stats", default=None)
            p.add_argument("--threads", type=int, default=1)  # accepted for compatibility (cli.py:279)
    args = ap.parse_args(argv)
    if args.cmd == "decode" and not (args.llr_in or args.infile):
        raise SystemExit("decode needs INFILE (coded bit file) or --llr-in")
    return _cmd_encode(args) if args.cmd == "encode" else _cmd_decode(args)


if __name__ == "__main__":
    sys.exit(main())
