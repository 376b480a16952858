"""In-tree build of libnysgpu.so (sm_100a only).

    python -m paper_2310_08333_b200.build        # or __graft_entry__.build()

Each ``csrc/*.cu`` is compiled with ``-gencode arch=compute_100a,code=sm_100a
-lineinfo`` and linked into ``paper_2310_08333_b200/libnysgpu.so`` next to
this file, so the built library travels to the GPU box with the repo snapshot.
"""

from __future__ import annotations

import concurrent.futures as cf
import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libnysgpu.so")
OBJ = os.path.join(HERE, "_obj")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O3",
    "--expt-relaxed-constexpr",
    "-I", os.path.join(ROOT, "include"),
]


def nvcc() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _needs(obj, src):
    if not os.path.exists(obj):
        return True
    t = os.path.getmtime(obj)
    deps = [src] + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cuh")]
    deps.append(os.path.join(ROOT, "include", "nysgpu.h"))
    return any(os.path.getmtime(d) > t for d in deps)


GEN = os.path.join(OBJ, "gen")
NVCC_FLAGS += ["-I", GEN]
# development library: the NYS_* A/B switches of csrc/ (common.cuh dev_env) are
# compiled in; rebuild with -f when toggling (objects are cached by mtime only)
if os.environ.get("NYS_DEV_SWITCHES") == "1":
    NVCC_FLAGS += ["-DNYS_DEV_SWITCHES"]


def build(verbose: bool = False, force: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    tables = os.path.join(GEN, "zig_tables.h")
    if force or not os.path.exists(tables):
        from .gen_tables import write_header

        write_header(tables)
    cc = nvcc()
    jobs = []
    objs = []
    for src in sources():
        obj = os.path.join(OBJ, os.path.basename(src)[:-3] + ".o")
        objs.append(obj)
        if force or _needs(obj, src):
            jobs.append([cc, *NVCC_FLAGS, "-c", src, "-o", obj])
    with cf.ThreadPoolExecutor(max_workers=min(8, max(1, len(jobs)))) as ex:
        for cmd, res in zip(jobs, ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), jobs)):
            if verbose or res.returncode != 0:
                sys.stderr.write(res.stdout + res.stderr)
            if res.returncode != 0:
                raise RuntimeError("nvcc failed: " + " ".join(cmd))
    if force or jobs or not os.path.exists(OUT):
        link = [cc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", OUT, *objs]
        res = subprocess.run(link, capture_output=True, text=True)
        if res.returncode != 0:
            sys.stderr.write(res.stdout + res.stderr)
            raise RuntimeError("link failed")
    return OUT


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
