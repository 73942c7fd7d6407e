"""Build libkvq.so in-tree with nvcc for sm_100a (called by __graft_entry__.build())."""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libkvq.so")
SOURCES = ["kvq_api.cu", "kvq_prefill.cu", "kvq_f16.cu", "kvq_calib.cu", "kvq_attend.cu", "kvq_attend_wa.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-ffp-contract=off", "-Xptxas", "-v"]
# diagnostics builds only (e.g. -DKVQ_TS_DEBUG: phase timestamps of the attend kernel)
FLAGS += os.environ.get("KVQ_EXTRA_NVCC_FLAGS", "").split()


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(HERE, "..", "include", "kvq.h")]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not stale():
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    objs = [os.path.join(CSRC, s[:-3] + f".{os.getpid()}.o") for s in SOURCES]
    cmds = [[NVCC, *FLAGS, "-c", "-o", o, os.path.join(CSRC, s)] for s, o in zip(SOURCES, objs)]
    # one nvcc per translation unit, in parallel, then one link
    with ThreadPoolExecutor(len(cmds)) as ex:
        rs = list(ex.map(lambda c: subprocess.run(c, capture_output=True, text=True), cmds))
    link = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o", tmp, *objs]
    log = os.path.join(HERE, "build.log")
    text = "".join(" ".join(c) + "\n" + r.stdout + r.stderr for c, r in zip(cmds, rs))
    ok = all(r.returncode == 0 for r in rs)
    if ok:
        rl = subprocess.run(link, capture_output=True, text=True)
        text += " ".join(link) + "\n" + rl.stdout + rl.stderr
        ok = rl.returncode == 0
    for o in objs:
        if os.path.exists(o):
            os.remove(o)
    with open(log, "w") as f:
        f.write(text)
    if not ok:
        sys.stderr.write(text[-8000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    os.replace(tmp, LIB)
    if verbose:
        print(text)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
