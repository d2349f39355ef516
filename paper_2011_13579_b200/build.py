"""Build the sm_100a extension library in-tree: libvitertile_b200.so.

Steps: generate the per-code ACS kernels (csrc/gen_kernels.py), compile each
translation unit with nvcc for sm_100a in parallel, link one shared library
exposing the C ABI of include/vitertile_b200.h.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(HERE, "_obj")
LIB = os.path.join(HERE, "libvitertile_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v"] + os.environ.get("VT_EXTRA_NVCC", "").split()


def _compile(src: str) -> tuple[str, str]:
    obj = os.path.join(OBJ, os.path.basename(src).replace(".cu", ".o"))
    stamp = obj + ".flags"  # the compile flags of the cached object (VT_EXTRA_NVCC changes force a rebuild)
    flags = " ".join(ARCH + FLAGS)
    same_flags = os.path.exists(stamp) and open(stamp).read() == flags
    if same_flags and os.path.exists(obj) and os.path.getmtime(obj) >= max(
            os.path.getmtime(src), *[os.path.getmtime(h) for h in glob.glob(os.path.join(CSRC, "*.cuh"))],
            *[os.path.getmtime(h) for h in glob.glob(os.path.join(CSRC, "gen", "*.inc"))],
            os.path.getmtime(os.path.join(HERE, "..", "include", "vitertile_b200.h"))):
        return obj, "(cached)"
    cmd = [NVCC, *ARCH, *FLAGS, "-c", "-o", obj, src]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    with open(stamp, "w") as fh:
        fh.write(flags)
    return obj, r.stderr


def build(verbose: bool = False) -> str:
    sys.path.insert(0, CSRC)
    try:
        import gen_kernels  # noqa: E402
    finally:
        sys.path.pop(0)
    os.makedirs(OBJ, exist_ok=True)
    gen_files = gen_kernels.generate(os.path.join(CSRC, "gen"))
    srcs = gen_files + [os.path.join(CSRC, "vt_capi.cu"), os.path.join(CSRC, "vt_channel.cu"),
                        os.path.join(CSRC, "vt_matrix_r4.cu"), os.path.join(CSRC, "vt_forward.cu"),
                        os.path.join(CSRC, "vt_tiles.cu")]
    with cf.ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as ex:
        results = list(ex.map(_compile, srcs))
    if verbose:
        for obj, log in results:
            lines = [ln for ln in log.splitlines() if "registers" in ln or "spill" in ln]
            print(os.path.basename(obj), " | ".join(ln.strip() for ln in lines))
    objs = [o for o, _ in results]
    newest = max(os.path.getmtime(o) for o in objs)
    if not os.path.exists(LIB) or os.path.getmtime(LIB) < newest:
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lcudart"]
        subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(verbose=True))
