"""In-tree build of the native library ``libhexbench_b200.so`` (sm_100a).

Each ``csrc/*.cu`` is compiled to an object in parallel, then linked into a
shared library next to this file, so the built ``.so`` travels with the repo
snapshot to the GPU box.  Rebuilds only when a source or header is newer than
the library.
"""

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build", "native")
LIB = os.path.join(HERE, "libhexbench_b200.so")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include")]


def _sources():
    return sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith(".cu"))


def _deps():
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)]
    deps.append(os.path.join(ROOT, "include", "hexbench_b200.h"))
    return deps


def up_to_date():
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(d) <= t for d in _deps())


def _compile(src, defines=(), build_dir=BUILD, extra=()):
    obj = os.path.join(build_dir, os.path.basename(src) + ".o")
    log = obj + ".ptxas.log"
    cmd = [NVCC, *ARCH, *FLAGS, *extra, *[f"-D{d}" for d in defines], "-c", src, "-o", obj]
    res = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as fh:
        fh.write(res.stdout + res.stderr)
    if res.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr[-6000:]}")
    return obj


def build(force=False, verbose=False, defines=(), lib=LIB, extra_flags=()):
    """Build the library (``defines``/``lib``/``extra_flags`` are for tuning
    experiments: variant builds go to a separate path and never replace the
    product)."""
    if not force and not defines and not extra_flags and lib == LIB and up_to_date():
        return LIB
    if defines or extra_flags:
        import hashlib
        tag = hashlib.sha1("|".join((*defines, *extra_flags)).encode()).hexdigest()[:12]
        build_dir = os.path.join(BUILD, "v_" + tag)
    else:
        build_dir = BUILD
    os.makedirs(build_dir, exist_ok=True)
    srcs = _sources()
    with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 4)) as pool:
        objs = list(pool.map(lambda s: _compile(s, defines, build_dir, extra_flags), srcs))
    tmp = lib + ".tmp"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static", "-lrt", "-ldl",
           "-lpthread"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr[-4000:]}")
    os.replace(tmp, lib)
    if verbose:
        print(f"built {lib}")
    return lib


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
