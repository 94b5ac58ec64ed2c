"""Build libnsreflector.so in-tree with nvcc for sm_100a (no JIT, no torch extension)."""
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libnsreflector.so")
SOURCES = ["ns_api.cu", "ns_fp64.cu", "ns_mixed.cu", "ns_reanchor.cu", "ns_shard.cu", "ns_small.cu", "ns_setup.cu", "ns_outer.cu", "ns_ozaki.cu"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def _nccl_dir():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (spec.submodule_search_locations if spec else []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("NCCL headers/library (nvidia-nccl) not found")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC", "-shared", "-Xptxas", "-v", "--expt-relaxed-constexpr"]


STAMP = LIB + ".sha256"


def _source_hash(cmd_tail):
    """sha256 over every source the library is built from (csrc/*, the public header) and the compile
    command: the staleness test (mtimes are not trusted -- a shipped .so newer than edited sources, or
    sources restored with old mtimes, must still rebuild)."""
    h = hashlib.sha256()
    deps = sorted(os.path.join(CSRC, f) for f in os.listdir(CSRC)) + [
        os.path.join(HERE, "..", "include", "nsreflector.h")]
    for d in deps:
        h.update(os.path.basename(d).encode())
        with open(d, "rb") as f:
            h.update(f.read())
    h.update(" ".join(cmd_tail).encode())
    return h.hexdigest()


def build(force=False, verbose=False):
    nccl = _nccl_dir()
    link = ["-I" + os.path.join(nccl, "include"), "-L" + os.path.join(nccl, "lib"), "-l:libnccl.so.2",
            "-Xlinker", "-rpath=" + os.path.join(nccl, "lib")]
    extra = os.environ.get("NS_NVCC_EXTRA", "").split()   # developer experiments (e.g. -DNS_OZ_A_TMEM=0)
    cmd = [NVCC] + FLAGS + extra + ["-o", LIB] + [os.path.join(CSRC, s) for s in SOURCES] + link
    digest = _source_hash(FLAGS + extra + SOURCES)
    if not force and os.path.exists(LIB) and os.path.exists(STAMP):
        with open(STAMP) as f:
            if f.read().strip() == digest:
                return LIB
    res = subprocess.run(cmd, capture_output=True, text=True)
    log = os.path.join(HERE, "build.log")
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libnsreflector.so (see %s)" % log)
    with open(STAMP, "w") as f:
        f.write(digest + "\n")
    if verbose:
        print(res.stderr)
    return LIB


if __name__ == "__main__":
    build(force=True, verbose=True)
