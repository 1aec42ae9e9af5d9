"""Build libfastlsh.so in-tree with nvcc for sm_100a (no JIT, no torch extension machinery)."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
OUT = os.path.join(HERE, "libfastlsh.so")
BUILD = os.path.join(HERE, "_build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = [*os.environ.get("FASTLSH_NVCC_EXTRA", "").split(), "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2", "--expt-relaxed-constexpr",
          "-I", os.path.join(ROOT, "include")]
SOURCES = ["api.cu", "gather.cu", "gather_inst0.cu", "gather_inst1.cu", "gather_inst2.cu", "gather_inst3.cu",
           "gather_tmem.cu", "tables.cu", "query.cu", "transforms.cu", "keys.cu", "e2lsh_tcgen05.cu", "packer.cpp",
           "gather_rows.cu", "gather_rows_inst0.cu", "gather_rows_inst1.cu", "gather_rows_inst2.cu",
           "gather_rows_inst3.cu", "gather_rows_inst4.cu", "gather_rows_inst5.cu", "rpacker.cpp", "jit.cpp", "probe.cu", "mc.cpp", "generic.cu"]


def _stale(out: str, deps) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def _deps(path: str, seen=None) -> list:
    """The file and every local header it includes (transitively)."""
    seen = set() if seen is None else seen
    if path in seen or not os.path.exists(path):
        return []
    seen.add(path)
    out = [path]
    for line in open(path):
        line = line.strip()
        if line.startswith("#include \""):
            inc = line.split('"')[1]
            out += _deps(os.path.normpath(os.path.join(os.path.dirname(path), inc)), seen)
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    objs, jobs = [], []
    for src in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or _stale(o, _deps(s)):
            lang = ["-x", "cu"] if src.endswith(".cu") else ["-x", "c++"]
            jobs.append([NVCC, *ARCH, *COMMON, *lang, "-c", s, "-o", o] +
                        (["-Xptxas", "-v"] if verbose and src.endswith(".cu") else []))
    if jobs:
        with ThreadPoolExecutor(max_workers=min(len(jobs), os.cpu_count() or 4)) as ex:
            results = list(ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs))
        for cmd, r in zip(jobs, results):
            if verbose and r.stderr:
                sys.stderr.write(r.stderr)
            if r.returncode != 0:
                raise RuntimeError(f"nvcc failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    if force or jobs or _stale(OUT, objs):
        link = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", OUT + ".tmp", *objs, "-lcuda", "-ldl"]
        r = subprocess.run(link, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"link failed: {' '.join(link)}\n{r.stdout}\n{r.stderr}")
        os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
