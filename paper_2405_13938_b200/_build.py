"""Build libexmy.so in-tree with nvcc for sm_100a (no JIT cache: the .so
travels with the repo snapshot to the GPU box)."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "libexmy.so")
BUILD = os.path.join(PKG, "build")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "-I", os.path.join(ROOT, "include"), "-I", CSRC]

# one translation unit per op family so they compile in parallel
UNITS = ["exmy_abi.cu", "exmy_tu_hist.cu", "exmy_tu_quant.cu", "exmy_tu_encode.cu", "exmy_tu_decode.cu",
         "exmy_tu_blk_encode.cu", "exmy_tu_blk_decode.cu", "exmy_tu_grouped.cu",
         "exmy_tu_fscale.cu", "exmy_tu_push.cu", "exmy_ckpt.cpp",
         "exmy_tu_bag.cu", "exmy_tu_probe.cu", "exmy_tu_gemv.cu"]
HEADERS = ["exmy_device.cuh", "exmy_kernels.cuh", "exmy_fast.cuh", "exmy_blocked.cuh", "exmy_launch.cuh", "exmy_grouped.cuh",
           "exmy_fscale.cuh", "exmy_tma.cuh", "exmy_narrow.cuh", "exmy_gemv.cuh"]


def _sources():
    return [os.path.join(CSRC, u) for u in UNITS]


def _deps():
    return _sources() + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "exmy.h")]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in _deps() if os.path.exists(p))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    log = []

    def compile_one(src):
        obj = os.path.join(BUILD, os.path.splitext(os.path.basename(src))[0] + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, "-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        log.append((src, r.stdout + r.stderr))
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        return obj

    with ThreadPoolExecutor(max_workers=len(UNITS)) as ex:
        objs = list(ex.map(compile_one, _sources()))
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    with open(os.path.join(BUILD, "ptxas.log"), "w") as f:
        for src, out in log:
            f.write(f"==== {src}\n{out}\n")
    if verbose:
        print(f"built {LIB}", file=sys.stderr)
    return LIB


def build_variant(out: str, extra: list[str], units=("exmy_tu_grouped.cu",)) -> str:
    """A/B builds: recompile `units` with extra nvcc flags (e.g. -DNAME=V) and
    link them with the main build's other objects into `out`."""
    build()
    vdir = os.path.join(BUILD, "variant_" + os.path.basename(out).replace(".so", ""))
    os.makedirs(vdir, exist_ok=True)
    objs = []
    for u in UNITS:
        if u in units:
            obj = os.path.join(vdir, os.path.splitext(u)[0] + ".o")
            r = subprocess.run([NVCC, *ARCH, *FLAGS, *extra, "-c", os.path.join(CSRC, u), "-o", obj],
                               capture_output=True, text=True)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {u}:\n{r.stderr}")
            with open(os.path.join(vdir, "ptxas.log"), "w") as f:
                f.write(r.stdout + r.stderr)
            objs.append(obj)
        else:
            objs.append(os.path.join(BUILD, os.path.splitext(u)[0] + ".o"))
    r = subprocess.run([NVCC, *ARCH, "-shared", "-o", out, *objs, "-lcudart"], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr}")
    return out


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
