"""Build libgfwa.so in-tree with nvcc for sm_100a (no JIT, no torch extension).

Each ``csrc/*.cu`` is compiled to an object in ``build/`` (in parallel), then
linked into ``paper_2512_07782_b200/libgfwa.so``.  Flags:
``-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17``.

``python _build.py --variant NAME -DX=Y ...`` builds an experiment variant into
``paper_2512_07782_b200/variants/libgfwa_NAME.so`` (select it at run time with
``GFWA_LIB=<path>``); the default library is unaffected.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build", "gfwa")
LIB = os.path.join(PKG, "libgfwa.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ARCH + [
    "-O3",
    "-lineinfo",
    "-std=c++17",
    "-Xcompiler",
    "-fPIC",
    "--expt-relaxed-constexpr",
    "-Xptxas",
    "-v",
    "-I",
    os.path.join(ROOT, "include"),
]

# per-file register caps: the tensor-core backward runs 10 warps / CTA (1 CTA/SM),
# so up to 200 registers per thread are available to its softmax warps (the
# forward moves registers between warpgroups with setmaxnreg instead)
PER_FILE = {"attn_tc_bwd.cu": ["-maxrregcount=200"]}


def _deps_mtime() -> float:
    files = glob.glob(os.path.join(CSRC, "*")) + glob.glob(os.path.join(ROOT, "include", "*.h"))
    return max(os.path.getmtime(f) for f in files)


def _compile(args) -> tuple[str, str]:
    src, bdir, extra = args
    obj = os.path.join(bdir, os.path.basename(src) + ".o")
    cmd = [NVCC, *FLAGS, *PER_FILE.get(os.path.basename(src), []), *extra, "-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr}")
    return obj, r.stderr


def build(force: bool = False, verbose: bool = False, extra: list[str] | None = None,
          variant: str | None = None) -> str:
    extra = list(extra or [])
    out = LIB if variant is None else os.path.join(PKG, "variants", f"libgfwa_{variant}.so")
    bdir = BUILD if variant is None else os.path.join(BUILD, "variants", variant)
    if not force and variant is None and os.path.exists(out) and os.path.getmtime(out) >= _deps_mtime():
        return out
    os.makedirs(bdir, exist_ok=True)
    os.makedirs(os.path.dirname(out), exist_ok=True)
    srcs = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    with cf.ThreadPoolExecutor(max_workers=min(8, len(srcs))) as ex:
        results = list(ex.map(_compile, [(s, bdir, extra) for s in srcs]))
    if verbose:
        for _, log in results:
            sys.stderr.write(log)
    tmp = out + f".tmp{os.getpid()}"
    # no -lcuda: driver entry points are resolved at run time (csrc/driver_api.cuh),
    # so the library also loads on hosts without a driver
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *[o for o, _ in results]]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    argv = sys.argv[1:]
    variant = None
    if "--variant" in argv:
        variant = argv[argv.index("--variant") + 1]
    defines = [a for a in argv if a.startswith("-D")]
    print(build(force="--force" in argv or variant is not None, verbose="-v" in argv, extra=defines,
                variant=variant))
