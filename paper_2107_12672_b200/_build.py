"""In-tree build of libddvr.so for sm_100a (nvcc cross-compiles without a GPU).

The kernels are split over several translation units (csrc/ddvr_*.cu sharing
csrc/ddvr_device.cuh) that compile in parallel and link into one shared
library with the static CUDA runtime.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
HDR = os.path.join(ROOT, "include", "ddvr.h")
OUT = os.path.join(HERE, "libddvr.so")
OBJ = os.path.join(ROOT, "build", "ddvr")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    return "nvcc"


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def stale(out: str = OUT) -> bool:
    """True when ``out`` is missing or older than any source it is built from."""
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    deps = sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [HDR, __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def _run(cmd):
    proc = subprocess.run(cmd, capture_output=True, text=True)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError(f"nvcc failed ({proc.returncode}): {' '.join(cmd)}")
    return proc.stderr


VARIANTS = os.path.join(HERE, "_variants")


def build_variant(name: str, defines) -> str:
    """Experiment build with extra -D switches into _variants/libddvr_<name>.so
    (select it at run time with DDVR_LIB=<path>); the product is build()."""
    return build(force=True, out=os.path.join(VARIANTS, f"libddvr_{name}.so"),
                 obj=os.path.join(OBJ, "v_" + name), extra=[f"-D{d}" for d in defines])


def build(force: bool = False, verbose: bool = False, out: str = OUT, obj: str = OBJ,
          extra=()) -> str:
    """Compile csrc/*.cu into libddvr.so next to this file; return its path."""
    if not force and not stale():
        return OUT
    OUT_, OBJ_ = out, obj
    os.makedirs(OBJ_, exist_ok=True)
    os.makedirs(os.path.dirname(OUT_), exist_ok=True)
    inc = ["-I", os.path.join(ROOT, "include"), "-I", CSRC, *extra]
    jobs = []
    for src in sources():
        o = os.path.join(OBJ_, os.path.basename(src)[:-3] + ".o")
        jobs.append((o, [nvcc(), *NVCC_FLAGS, "-Xptxas", "-v", *inc, "-c", "-o", o, src]))
    with ThreadPoolExecutor(max_workers=max(1, min(len(jobs), os.cpu_count() or 1))) as ex:
        logs = list(ex.map(lambda j: _run(j[1]), jobs))
    if verbose:
        sys.stderr.write("".join(logs))
    _run([nvcc(), *ARCH, "-shared", "-o", OUT_ + ".tmp", *[o for o, _ in jobs]])
    os.replace(OUT_ + ".tmp", OUT_)
    return OUT_


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
