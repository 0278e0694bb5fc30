"""Builds libcvq_b200.so (sm_100a) in-tree with nvcc.

`python -m paper_2506_18879_b200.build` or `build()`; no JIT cache, the .so
travels with the repo snapshot to the GPU box.
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libcvq_b200.so")
SOURCES = ["capi.cu", "attn.cu", "attn_fast.cu", "attn_tc.cu", "attn_sp.cu", "encode.cu", "pack.cu", "train.cu", "train_value.cu", "mgpu.cu", "naive.cu", "decode.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-std=c++17", "-O3", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-fvisibility=hidden", "-shared", "-cudart", "static",
    "--expt-relaxed-constexpr", "-Xptxas", "-v", "-I" + os.path.join(ROOT, "include"), "-ldl",
]


def _extra():
    return os.environ.get("CVQ_NVCC_EXTRA", "").split()  # experiments, e.g. -DNAME=1


def _stale():
    if not os.path.exists(SO):
        return True
    try:  # a build with other experiment flags is stale too
        with open(SO + ".flags") as f:
            if f.read() != " ".join(_extra()):
                return True
    except OSError:
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [
        os.path.join(ROOT, "include", "cvq.h"), __file__]
    return any(os.path.getmtime(p) > t for p in deps)


def build(force=False, verbose=False):
    if not force and not _stale():
        return SO
    extra = _extra()
    cmd = [NVCC] + FLAGS + extra + ["-o", SO] + [os.path.join(CSRC, s) for s in SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        sys.stderr.write(r.stderr[-8000:])
        raise RuntimeError(f"nvcc failed (see {log})")
    with open(SO + ".flags", "w") as f:
        f.write(" ".join(extra))
    if verbose:
        sys.stderr.write(r.stderr)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
