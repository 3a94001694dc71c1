"""Build libtm.so (the C-ABI library) in-tree with nvcc for sm_100a.

    python -m paper_2506_03099_b200.build [--force]

Objects are compiled in parallel into csrc/build/ and linked into
paper_2506_03099_b200/libtm.so (git-ignored; travels to the GPU box).
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libtm.so")
BUILD = os.path.join(CSRC, "build")
ROOT = os.path.dirname(PKG)

SOURCES = ["api.cpp", "comm.cpp", "fmha_sm100.cu", "fmha_fp32.cu", "elementwise.cu", "peer.cu"]
HEADERS = ["ptx.cuh", "internal.h", "comm.h", "ulysses_map.h", "peer.cuh", "peer_map.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for p in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if p and os.path.exists(p):
            return p
    raise RuntimeError("nvcc not found")


def _nccl_default() -> str:
    try:
        import nvidia.nccl  # type: ignore
        base = list(nvidia.nccl.__path__)[0]
        cand = os.path.join(base, "lib", "libnccl.so.2")
        return cand if os.path.exists(cand) else ""
    except Exception:
        return ""


def _flags():
    tb = os.environ.get("TM_TRACE_BUILD")
    extra = {"1": ["-DTM_TRACE_ENABLED"], "spans": ["-DTM_SPANS_ENABLED"]}.get(tb, [])
    # TM_EXTRA_DEFINES="A=1 B": tuning variants for tools/ A/B builds only
    extra += ["-D" + d for d in os.environ.get("TM_EXTRA_DEFINES", "").split()]
    return extra + ARCH + ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC",
                   "-Xptxas", "-v", f"-I{os.path.join(ROOT, 'include')}",
                   f'-DTM_NCCL_DEFAULT="{_nccl_default()}"']


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "tm.h"),
                                                     os.path.abspath(__file__)]
    stamp = os.path.join(BUILD, "flags.txt")
    flags_now = " ".join(_flags())
    if not os.path.exists(stamp) or open(stamp).read() != flags_now:
        force = True
        with open(stamp, "w") as f:
            f.write(flags_now)
    objs, jobs = [], []
    for s in SOURCES:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + hdrs):
            jobs.append((src, obj))

    def compile_one(job):
        src, obj = job
        cmd = [nvcc()] + _flags() + ["-c", src, "-o", obj]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        return src, r.stderr

    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for src, log in ex.map(compile_one, jobs):
            if verbose:
                print(f"[tm build] {os.path.basename(src)}\n{log}", file=sys.stderr)
    if force or jobs or _stale(OUT, objs):
        tmp = OUT + f".tmp{os.getpid()}"
        cmd = [nvcc()] + ARCH + ["-shared", "-Xcompiler", "-fPIC", "-o", tmp] + objs + ["-ldl"]
        subprocess.check_call(cmd)
        os.replace(tmp, OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
