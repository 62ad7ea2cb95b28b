"""Compile the sm_100a solver library in-tree (``paper_2011_04240_b200/_swarm_am.so``).

Plain nvcc, no torch extension machinery: the library exports a C ABI
(include/swarm_am.h) and links the CUDA runtime statically, so the same
``.so`` is loadable from ctypes, cgo or JNI alike.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "_swarm_am.so")
# capi.cu holds the host side; the kernel variants are explicitly instantiated in inst_*.cu
# so the (independent, slow) device compilations run in parallel
SOURCES = [os.path.join(CSRC, f) for f in ("capi.cu", "inst_nb1_12.cu", "inst_nb1_16.cu", "inst_nb2.cu",
                                           "inst_nb48.cu", "inst_f32_nb1.cu", "inst_f32_nb248.cu",
                                           "inst_large.cu", "collisions.cu", "report.cu")]
DEPS = SOURCES + [os.path.join(CSRC, "am_kernel.cuh"), os.path.join(CSRC, "am_large.cuh"),
                  os.path.join(ROOT, "include", "swarm_am.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
]
LINK_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-shared", "--cudart", "static"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    return "nvcc"


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(d) > t for d in DEPS)


def build(force: bool = False, verbose: bool = False, extra_flags=()) -> str:
    if not force and not stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor
    import hashlib
    tag = hashlib.sha1(" ".join(extra_flags).encode()).hexdigest()[:8] if extra_flags else ""
    objdir = os.path.join(CSRC, "obj" + ("_" + tag if tag else ""))
    os.makedirs(objdir, exist_ok=True)
    log = os.path.join(HERE, "csrc", "build.log")

    headers = [d for d in DEPS if d not in SOURCES]

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src) + ".o")
        cmd = [nvcc(), *NVCC_FLAGS, *extra_flags, "-c", "-o", obj, src]
        # incremental: an object newer than its source and every shared header is reused
        # (A/B builds with extra flags keep their objects in their own directory)
        if not force and os.path.exists(obj) and \
                all(os.path.getmtime(obj) > os.path.getmtime(d) for d in [src, *headers]):
            return cmd, obj, subprocess.CompletedProcess(cmd, 0, "", "(up to date)\n")
        return cmd, obj, subprocess.run(cmd, capture_output=True, text=True)

    with ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        results = list(ex.map(compile_one, SOURCES))
    text = ""
    for cmd, obj, res in results:
        text += " ".join(cmd) + "\n" + res.stdout + res.stderr
    tmp = LIB + ".tmp"
    link = [nvcc(), *LINK_FLAGS, "-o", tmp, *[obj for _, obj, _ in results]]
    lres = None
    if all(res.returncode == 0 for _, _, res in results):
        lres = subprocess.run(link, capture_output=True, text=True)
        text += " ".join(link) + "\n" + lres.stdout + lres.stderr
    with open(log, "w") as fh:
        fh.write(text)
    if lres is None or lres.returncode != 0:
        sys.stderr.write(text[-4000:])
        raise RuntimeError(f"nvcc failed; see {log}")
    os.replace(tmp, LIB)
    if verbose:
        sys.stdout.write(text)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
