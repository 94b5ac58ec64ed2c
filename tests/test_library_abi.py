"""CPU-side checks of the C-ABI boundary: the library builds, loads and exports every symbol
include/nsreflector.h declares; host-side argument validation (no GPU needed: validation
happens before any CUDA call)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2605_24840_b200 import build
    build.build()
    import paper_2605_24840_b200 as nsr
    return nsr.load_library()


def _declared_symbols():
    with open(os.path.join(ROOT, "include", "nsreflector.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"\b(ns_[a-z_0-9]+)\s*\(", src)))


def test_header_symbols_exported(lib):
    import paper_2605_24840_b200 as nsr
    declared = _declared_symbols()
    assert set(declared) == set(nsr.EXPORTED_SYMBOLS)
    for name in declared:
        assert hasattr(lib, name), name


def test_build_info_names_target(lib):
    assert b"sm_100a" in lib.ns_build_info()


def test_workspace_sizes(lib):
    # 3 padded FP64 matrices dominate; d=16384 -> 3 * 2 GiB plus small tails (partials, tile lists incl.
    # the host entry's chunk-ordered copy of the first square's list: < 2 MiB)
    w = lib.ns_workspace_bytes(16384, 0)
    assert 3 * 16384 * 16384 * 8 <= w < 3 * 16384 * 16384 * 8 + (2 << 20)
    assert lib.ns_workspace_bytes(100, 0) >= 3 * 128 * 128 * 8      # padded to 128
    assert lib.ns_workspace_bytes_batched(256, 10, 0) >= 10 * 3 * 256 * 256 * 8
    assert lib.ns_workspace_bytes(0, 0) == 0


def test_argument_validation(lib):
    import paper_2605_24840_b200 as nsr
    res = nsr.NsResult()
    buf = ctypes.create_string_buffer(1 << 16)
    ws = ctypes.c_void_p((ctypes.addressof(buf) + 255) & ~255)
    fake = ctypes.c_void_p(0x1000)

    def call(d=64, ldh=64, s=0.0, alpha=1.0, k=3, max_steps=10, tol=1e-12, tm=0, prec=0, R=ctypes.c_void_p(0x2000),
             ldr=64, ws_bytes=1 << 30):
        return lib.ns_reflector(fake, d, ldh, s, alpha, k, max_steps, tol, tm, prec, R, ldr, ws, ws_bytes, None,
                                ctypes.byref(res))

    assert call(d=0) == 1
    assert call(ldh=10) == 1
    assert call(alpha=-1.0) == 1                 # (alpha = 0 selects the device Gershgorin bound)
    assert call(alpha=float("nan")) == 1
    assert call(s=float("inf")) == 1
    assert call(k=-1) == 1 and call(k=65) == 1
    assert call(max_steps=-1) == 1
    assert call(tol=-1.0) == 1
    assert call(tm=7) == 1
    assert call(prec=7) == 1                     # unknown precision
    assert call(prec=3, d=70000, ldh=70000, ldr=70000, k=3) == 1   # d <= 65536 on every path (Ozaki chunks INT32 sums)
    assert call(R=fake) == 1                     # aliasing
    assert call(ws_bytes=10) == 4                # NS_ERR_WORKSPACE
    assert b"workspace" in lib.ns_last_error()
    assert lib.ns_status_string(4) == b"NS_ERR_WORKSPACE"


def test_product_path_has_no_oracle_or_fallback():
    """The product package must not import the oracle nor contain a CPU fallback."""
    pkg = os.path.join(ROOT, "paper_2605_24840_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                with open(os.path.join(dirpath, fn)) as f:
                    src = f.read()
                assert "oracle" not in src.replace("oracle/", ""), fn
                assert "import numpy.linalg" not in src and "np.linalg" not in src, fn


def test_batched_result_records_are_a_sequence_of_dicts():
    """The batched entries return their per-problem records as a sequence that builds each dict on access
    (marshalling only: no arithmetic); it indexes, slices, iterates and compares like the list of dicts it replaces."""
    import paper_2605_24840_b200 as nsr
    n = 5
    raw = (nsr.NsResult * n)()
    for i in range(n):
        raw[i].steps, raw[i].flags, raw[i].index_cert, raw[i].residual = i + 1, 1, 7 - i, 0.5 * i
    outs = nsr._ResultList(raw)
    assert len(outs) == n and outs[2]["steps"] == 3 and outs[-1]["cert"] == 3
    assert [o["steps"] for o in outs] == [1, 2, 3, 4, 5]
    assert outs[1:3] == [outs[1], outs[2]] and isinstance(outs[1:3], list)
    assert outs == list(outs) and outs == nsr._ResultList(raw)
    other = (nsr.NsResult * n)()
    assert outs != nsr._ResultList(other)
    assert outs.column("steps").tolist() == [1, 2, 3, 4, 5] and outs.column("cert").tolist() == [7, 6, 5, 4, 3]
    with pytest.raises(IndexError):
        outs[n]
