"""Build libnsrgs.so in-tree with nvcc for sm_100a (no torch JIT cache involved).

    python -m paper_2604_07372_b200.build [-v]
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libnsrgs.so")
BUILD = os.path.join(PKG, "_build")
# "file@MACRO=v": the same source compiled once per value (wide_tc.cu: its block sizes are split over
# four objects, a single nvcc run over all of them takes > 8 minutes)
SOURCES = ["panel.cu", "sym.cu", "wide.cu", "wide_tc.cu@NSRGS_TC_PART=0", "wide_tc.cu@NSRGS_TC_PART=1",
           "wide_tc.cu@NSRGS_TC_PART=2", "wide_tc.cu@NSRGS_TC_PART=3", "bsr.cu", "polar.cu", "aux.cu", "objective64.cu", "probe.cu", "runtime.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
         "-I" + os.path.join(ROOT, "include"), "-I" + CSRC]


def _nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def _stale(obj: str, deps) -> bool:
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    return any(os.path.getmtime(d) > t for d in deps)


def _includes(path: str, seen=None) -> set:
    """Quoted #include files of `path`, recursively (the object's header dependencies)."""
    seen = set() if seen is None else seen
    with open(path) as f:
        for line in f:
            line = line.strip()
            if line.startswith("#include") and '"' in line:
                dep = os.path.normpath(os.path.join(os.path.dirname(path), line.split('"')[1]))
                if dep not in seen and os.path.exists(dep):
                    seen.add(dep)
                    _includes(dep, seen)
    return seen


def build(verbose: bool = False, force: bool = False, ptxas_v: bool = False) -> str:
    nvcc = _nvcc()
    os.makedirs(BUILD, exist_ok=True)
    jobs = []
    for item in SOURCES:
        src, _, macro = item.partition("@")
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, item.replace("@", ".").replace("=", "_") + ".o")
        if force or _stale(o, [s] + sorted(_includes(s))):
            cmd = [nvcc, *ARCH, *FLAGS, *(["-D" + macro] if macro else []), "-c", s, "-o", o]
            if ptxas_v:
                cmd += ["-Xptxas", "-v"]
            jobs.append(cmd)

    def run(cmd):
        r = subprocess.run(cmd, capture_output=True, text=True)
        return cmd, r

    with cf.ThreadPoolExecutor(max_workers=len(jobs) or 1) as ex:
        for cmd, r in ex.map(run, jobs):
            if verbose or r.returncode != 0:
                sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed for {cmd[-3]}")
    objs = [os.path.join(BUILD, s.replace("@", ".").replace("=", "_") + ".o") for s in SOURCES]
    if force or jobs or _stale(OUT, objs):
        cmd = [nvcc, *ARCH, "-shared", "-o", OUT, *objs, "-ldl"]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if verbose or r.returncode != 0:
            sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        if r.returncode != 0:
            raise RuntimeError("link of libnsrgs.so failed")
    return OUT


if __name__ == "__main__":
    build(verbose="-v" in sys.argv, force="-f" in sys.argv, ptxas_v="--ptxas" in sys.argv)
    print(OUT)
