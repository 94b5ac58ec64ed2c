"""Build a variant of libnsreflector.so with extra nvcc flags to another path (A/B experiments).

    python tools/build_variant.py build_ab/v0.so -DNS_SMALL_V2=0
then  python tools/ab_lib.py build_ab/v0.so tools/small_prof.py 2000
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_24840_b200 import build as b  # noqa: E402

out = os.path.abspath(sys.argv[1])
os.makedirs(os.path.dirname(out), exist_ok=True)
nccl = b._nccl_dir()
link = ["-I" + os.path.join(nccl, "include"), "-L" + os.path.join(nccl, "lib"), "-l:libnccl.so.2",
        "-Xlinker", "-rpath=" + os.path.join(nccl, "lib")]
cmd = [b.NVCC] + b.FLAGS + sys.argv[2:] + ["-o", out] + [os.path.join(b.CSRC, s) for s in b.SOURCES] + link
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode != 0:
    sys.stderr.write(r.stderr)
    sys.exit(1)
print(out)
