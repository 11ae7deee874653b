"""Build libpsd.so (all csrc/*.cu + *.cpp) for sm_100a, in-tree.

    python -m paper_2603_18016_b200.build_native

nvcc cross-compiles without a GPU, so this runs in the build container; the
resulting .so travels with the repo snapshot to the GPU box.
"""

from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libpsd.so")
BUILD = os.path.join(HERE, "csrc", "_build" + ("_exp" if os.environ.get("PSD_EXPERIMENTAL",
                                                                        "0") == "1" else ""))

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
         "-Xptxas", "-v", "-I", os.path.join(HERE, "..", "include")]


# PSD_EXPERIMENTAL=1 also builds the parked variants declared in
# include/psd_experimental.h (fused k-step draft decode, pre-tiled weight GEMM)
EXPERIMENTAL = os.environ.get("PSD_EXPERIMENTAL", "0") == "1"
EXPERIMENTAL_ONLY = {"decode_mk.cu"}
if EXPERIMENTAL:
    FLAGS = FLAGS + ["-DPSD_EXPERIMENTAL=1"]


def _sources():
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")) + glob.glob(os.path.join(CSRC, "*.cpp")))
    return [s for s in srcs if EXPERIMENTAL or os.path.basename(s) not in EXPERIMENTAL_ONLY]


def _needs(obj: str, src: str, headers: list[str]) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(f) > t for f in [src] + headers)


def build(verbose: bool = False, jobs: int = 8) -> str:
    os.makedirs(BUILD, exist_ok=True)
    headers = (glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))
               + glob.glob(os.path.join(HERE, "..", "include", "*.h")))
    procs = []
    objs = []
    for src in _sources():
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        objs.append(obj)
        if _needs(obj, src, headers):
            cmd = [NVCC] + ARCH + FLAGS + ["-c", src, "-o", obj]
            procs.append((src, subprocess.Popen(cmd, stdout=subprocess.PIPE,
                                                stderr=subprocess.STDOUT, text=True)))
        while len([p for _, p in procs if p.poll() is None]) >= jobs:
            procs[0][1].wait()
    for src, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            sys.stderr.write(out)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stdout.write(out)
    # relink when an object changed or the object set did (experimental switch)
    stamp = os.path.join(BUILD, "..", "_link_objs.txt")
    want = "\n".join(objs)
    have = open(stamp).read() if os.path.exists(stamp) else ""
    if (have != want or not os.path.exists(OUT)
            or any(os.path.getmtime(o) > os.path.getmtime(OUT) for o in objs)):
        cmd = [NVCC] + ARCH + ["-shared", "-o", OUT] + objs
        subprocess.run(cmd, check=True)
        with open(stamp, "w") as fh:
            fh.write(want)
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
