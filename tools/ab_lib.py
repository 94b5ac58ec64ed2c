"""A/B helper: run a script against another build of libnsreflector.so.

    python tools/ab_lib.py <path/to/libnsreflector.so> bench.py --steps 3 --warmup 3
"""
import os
import runpy
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_24840_b200 as nsr  # noqa: E402

nsr.load_library(os.path.abspath(sys.argv[1]))
sys.argv = sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
