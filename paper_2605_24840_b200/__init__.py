"""Thin ctypes binding of libnsreflector.so (include/nsreflector.h).

Argument marshalling only: every step of the Newton–Schulz path runs in the CUDA
kernels of the shared library.  torch is used for device memory and streams.  There
is no CPU fallback: importing this package on a machine without the built library
raises, and calling it with CPU tensors raises.
"""
import collections.abc
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libnsreflector.so")

NS_PREC_FP64, NS_PREC_MIXED_BF16X3, NS_PREC_MIXED_TF32X3, NS_PREC_FP64_OZAKI = 0, 1, 2, 3
NS_TOL_ABS, NS_TOL_PER_SQRT_D = 0, 1
NS_OK = 0
NS_F_CONVERGED, NS_F_MAX_STEPS, NS_F_INDEX_MISMATCH = 1, 2, 4
NS_F_SCALING_SUSPECT, NS_F_NONFINITE, NS_F_SHIFT_ON_SPECTRUM = 8, 16, 32

EXPORTED_SYMBOLS = (
    "ns_workspace_bytes", "ns_workspace_bytes_batched", "ns_workspace_bytes_host", "ns_reflector",
    "ns_reflector_host", "ns_reflector_batched", "ns_symm_product", "ns_build_info", "ns_status_string",
    "ns_last_error", "ns_profile_enable", "ns_profile_reset", "ns_profile_get", "ns_options_default",
    "ns_reflector_ex", "ns_comm_get_unique_id", "ns_comm_init", "ns_comm_destroy", "ns_shard_plan",
    "ns_workspace_bytes_sharded", "ns_reflector_sharded", "ns_shard_chunks", "ns_workspace_bytes_setup", "ns_scale_bound",
    "ns_shift_certificate", "ns_workspace_bytes_alg1", "ns_alg1_rotated_quartic", "ns_alg1_rotated_quartic_ex",
    "ns_debug_mx_trace",
    "ns_symm_product_shard", "ns_workspace_bytes_sharded_emulated", "ns_reflector_sharded_emulated",
    "ns_comm_init_host", "ns_shard_rows", "ns_reflector_sharded_rows", "ns_reflector_batched_dev",
    "ns_workspace_bytes_inertia", "ns_inertia", "ns_shift_bisect", "ns_workspace_bytes_ex", "ns_debug_small_trace", "ns_debug_p64_trace",
)


class NsResult(ctypes.Structure):
    _fields_ = [("steps", ctypes.c_int32), ("flags", ctypes.c_int32), ("residual", ctypes.c_double),
                ("trace", ctypes.c_double), ("index_cert", ctypes.c_int64), ("kernel_launches", ctypes.c_int32),
                ("switch_step", ctypes.c_int32), ("pre_polish_residual", ctypes.c_double), ("alpha", ctypes.c_double)]

    def as_dict(self):
        return dict(steps=self.steps, flags=self.flags, residual=self.residual, trace=self.trace,
                    cert=self.index_cert, launches=self.kernel_launches, switch_step=self.switch_step,
                    pre_polish_residual=self.pre_polish_residual, alpha=self.alpha)


class _ResultList(collections.abc.Sequence):
    """Per-problem result records of a batched call, converted to dicts on access (building thousands of dicts
    eagerly cost ~4 ms per configs[1] call -- marshalling, so it stays out of the call)."""

    def __init__(self, arr):
        self._arr = arr

    def __len__(self):
        return len(self._arr)

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self._arr[j].as_dict() for j in range(*i.indices(len(self._arr)))]
        return self._arr[i].as_dict()

    def __eq__(self, other):
        if isinstance(other, (_ResultList, list, tuple)):
            return len(self) == len(other) and all(a == b for a, b in zip(self, other))
        return NotImplemented

    def __repr__(self):
        return repr(list(self))

    def column(self, name):
        """One field of every record as a numpy array (steps, flags, residual, trace, cert, ...)."""
        field = {"cert": "index_cert", "launches": "kernel_launches"}.get(name, name)
        return np.array([getattr(r, field) for r in self._arr])


class NsOptions(ctypes.Structure):
    _fields_ = [("switch_tol", ctypes.c_double), ("cg_iters", ctypes.c_int32), ("stop_at_switch", ctypes.c_int32),
                ("lookahead", ctypes.c_int32), ("polish", ctypes.c_int32), ("reserved", ctypes.c_int32 * 2),
                ("filter_a", ctypes.c_double), ("filter_b", ctypes.c_double), ("filter_c", ctypes.c_double * 3)]


class NsProfile(ctypes.Structure):
    _fields_ = [("n_square", ctypes.c_int64), ("n_update", ctypes.c_int64), ("ms_square", ctypes.c_double),
                ("ms_update", ctypes.c_double), ("n_calls", ctypes.c_int64),
                ("n_lowp", ctypes.c_int64), ("ms_lowp", ctypes.c_double), ("lowp_flops", ctypes.c_double),
                ("n_oz", ctypes.c_int64), ("ms_oz", ctypes.c_double), ("oz_ops", ctypes.c_double)]


class NsShiftCert(ctypes.Structure):
    _fields_ = [("margin_hat", ctypes.c_double), ("margin_lb", ctypes.c_double), ("reuse_margin_lb", ctypes.c_double),
                ("midpoint", ctypes.c_double), ("admissible", ctypes.c_int32), ("reuse_ok", ctypes.c_int32),
                ("midpoint_ok", ctypes.c_int32), ("pad", ctypes.c_int32)]


class NsAlg1Result(ctypes.Structure):
    _fields_ = [("iters", ctypes.c_int32), ("morse_index", ctypes.c_int32), ("success", ctypes.c_int32),
                ("stop_reason", ctypes.c_int32), ("grad_norm", ctypes.c_double), ("refreshes", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("s_last", ctypes.c_double)]


class NsAlg1Policy(ctypes.Structure):
    _fields_ = [("policy", ctypes.c_int32), ("pad", ctypes.c_int32), ("damp", ctypes.c_double),
                ("clip", ctypes.c_double), ("reuse_margin", ctypes.c_double), ("eps", ctypes.c_double)]


NS_SHIFT_POLICIES = {"midpoint": 0, "damped": 1, "reuse_refresh": 2}


class NsBisect(ctypes.Structure):
    _fields_ = [("s", ctypes.c_double), ("lam_k_lo", ctypes.c_double), ("lam_k_hi", ctypes.c_double),
                ("lam_k1_lo", ctypes.c_double), ("lam_k1_hi", ctypes.c_double), ("eps", ctypes.c_double),
                ("alpha", ctypes.c_double), ("probes", ctypes.c_int32), ("unresolved", ctypes.c_int32),
                ("ok", ctypes.c_int32), ("pad", ctypes.c_int32)]


class NsError(RuntimeError):
    pass


# int allgather(const void* send, void* recv, size_t bytes, void* user)   (ns_host_allgather_fn)
HOST_ALLGATHER = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p)
_HOST_CALLBACKS = {}     # comm handle value -> CFUNCTYPE object (kept alive while the communicator exists)


_lib = None


def load_library(path=LIB_PATH):
    """Load libnsreflector.so (raises if it was not built -- there is no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise NsError(f"{path} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(path)
    c_i64, c_i32, c_dbl, c_vp, c_sz = ctypes.c_int64, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p, ctypes.c_size_t
    lib.ns_workspace_bytes.restype = c_sz
    lib.ns_workspace_bytes.argtypes = [c_i64, ctypes.c_int]
    lib.ns_workspace_bytes_batched.restype = c_sz
    lib.ns_workspace_bytes_batched.argtypes = [c_i64, c_i64, ctypes.c_int]
    lib.ns_workspace_bytes_host.restype = c_sz
    lib.ns_workspace_bytes_host.argtypes = [c_i64, ctypes.c_int]
    lib.ns_reflector.restype = ctypes.c_int
    lib.ns_reflector.argtypes = [c_vp, c_i64, c_i64, c_dbl, c_dbl, c_i32, c_i32, c_dbl, ctypes.c_int, ctypes.c_int,
                                 c_vp, c_i64, c_vp, c_sz, c_vp, ctypes.POINTER(NsResult)]
    lib.ns_reflector_ex.restype = ctypes.c_int
    lib.ns_reflector_ex.argtypes = [c_vp, c_i64, c_i64, c_dbl, c_dbl, c_i32, c_i32, c_dbl, ctypes.c_int, ctypes.c_int,
                                    c_vp, c_i64, c_vp, c_sz, c_vp, ctypes.POINTER(NsOptions), ctypes.POINTER(NsResult)]
    lib.ns_options_default.restype = None
    lib.ns_options_default.argtypes = [ctypes.POINTER(NsOptions)]
    lib.ns_reflector_host.restype = ctypes.c_int
    lib.ns_reflector_host.argtypes = lib.ns_reflector.argtypes
    lib.ns_reflector_batched.restype = ctypes.c_int
    lib.ns_reflector_batched.argtypes = [c_vp, c_i64, c_i64, c_i64, c_vp, c_vp, c_vp, c_i32, c_dbl, ctypes.c_int,
                                         ctypes.c_int, c_vp, c_i64, c_vp, c_sz, c_vp, ctypes.POINTER(NsResult)]
    lib.ns_symm_product.restype = ctypes.c_int
    lib.ns_symm_product.argtypes = [c_vp, c_vp, c_vp, c_i64, c_i64, c_i32, ctypes.c_int, c_vp, c_sz, c_vp]
    lib.ns_workspace_bytes_sharded_emulated.restype = c_sz
    lib.ns_workspace_bytes_sharded_emulated.argtypes = [c_i64, ctypes.c_int]
    lib.ns_reflector_sharded_emulated.restype = ctypes.c_int
    lib.ns_reflector_sharded_emulated.argtypes = [c_i32, c_vp, c_i64, c_i64, c_dbl, c_dbl, c_i32, c_i32, c_dbl,
                                                  ctypes.c_int, c_vp, c_i64, c_vp, c_sz, c_vp, c_i32, c_vp]
    lib.ns_workspace_bytes_ex.restype = c_sz
    lib.ns_workspace_bytes_ex.argtypes = [c_i64, ctypes.c_int, ctypes.POINTER(NsOptions)]
    lib.ns_reflector_batched_dev.restype = ctypes.c_int
    lib.ns_reflector_batched_dev.argtypes = lib.ns_reflector_batched.argtypes
    lib.ns_workspace_bytes_inertia.restype = c_sz
    lib.ns_workspace_bytes_inertia.argtypes = [c_i64, ctypes.c_int]
    lib.ns_inertia.restype = ctypes.c_int
    lib.ns_inertia.argtypes = [c_vp, c_i64, c_i64, c_dbl, ctypes.c_int, c_i32, c_vp, c_sz, c_vp,
                               ctypes.POINTER(c_i64), ctypes.POINTER(c_i32), ctypes.POINTER(NsResult)]
    lib.ns_shift_bisect.restype = ctypes.c_int
    lib.ns_shift_bisect.argtypes = [c_vp, c_i64, c_i64, c_i32, c_dbl, c_dbl, c_dbl, c_i32, ctypes.c_int, c_vp, c_sz,
                                    c_vp, ctypes.POINTER(NsBisect)]
    lib.ns_comm_init_host.restype = ctypes.c_int
    lib.ns_comm_init_host.argtypes = [ctypes.c_int, ctypes.c_int, HOST_ALLGATHER, c_vp, ctypes.POINTER(c_vp)]
    lib.ns_shard_rows.restype = ctypes.c_int
    lib.ns_shard_rows.argtypes = [c_i64, ctypes.c_int, ctypes.c_int, ctypes.POINTER(c_i64), ctypes.POINTER(c_i64)]
    lib.ns_reflector_sharded_rows.restype = ctypes.c_int
    lib.ns_reflector_sharded_rows.argtypes = [c_vp, c_vp, c_i64, c_i64, c_dbl, c_dbl, c_i32, c_i32, c_dbl,
                                              ctypes.c_int, ctypes.c_int, c_vp, c_i64, c_vp, c_sz, c_vp,
                                              ctypes.POINTER(NsResult)]
    lib.ns_symm_product_shard.restype = ctypes.c_int
    lib.ns_symm_product_shard.argtypes = [c_vp, c_vp, c_vp, c_i32, c_i64, c_i32, c_i32, c_i32, c_vp, c_sz, c_vp]
    lib.ns_build_info.restype = ctypes.c_char_p
    lib.ns_status_string.restype = ctypes.c_char_p
    lib.ns_status_string.argtypes = [ctypes.c_int]
    lib.ns_last_error.restype = ctypes.c_char_p
    lib.ns_profile_enable.argtypes = [ctypes.c_int]
    lib.ns_profile_enable.restype = None
    lib.ns_profile_reset.restype = None
    lib.ns_profile_get.argtypes = [ctypes.POINTER(NsProfile)]
    lib.ns_profile_get.restype = None
    lib.ns_comm_get_unique_id.restype = ctypes.c_int
    lib.ns_comm_get_unique_id.argtypes = [ctypes.c_char_p]
    lib.ns_comm_init.restype = ctypes.c_int
    lib.ns_comm_init.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_char_p, ctypes.POINTER(c_vp)]
    lib.ns_comm_destroy.restype = ctypes.c_int
    lib.ns_comm_destroy.argtypes = [c_vp]
    lib.ns_shard_plan.restype = ctypes.c_int
    lib.ns_shard_plan.argtypes = [c_i64, ctypes.c_int, ctypes.c_int, c_vp, c_i32, ctypes.POINTER(c_i32)]
    lib.ns_shard_chunks.restype = ctypes.c_int
    lib.ns_shard_chunks.argtypes = [c_i64, ctypes.c_int, ctypes.POINTER(c_i32), ctypes.POINTER(c_i32)]
    lib.ns_workspace_bytes_sharded.restype = c_sz
    lib.ns_workspace_bytes_sharded.argtypes = [c_i64, ctypes.c_int]
    lib.ns_reflector_sharded.restype = ctypes.c_int
    lib.ns_reflector_sharded.argtypes = [c_vp, c_vp, c_i64, c_i64, c_dbl, c_dbl, c_i32, c_i32, c_dbl, ctypes.c_int,
                                         c_vp, c_i64, c_vp, c_sz, c_vp, ctypes.POINTER(NsResult)]
    lib.ns_workspace_bytes_setup.restype = c_sz
    lib.ns_workspace_bytes_setup.argtypes = [c_i64]
    lib.ns_scale_bound.restype = ctypes.c_int
    lib.ns_scale_bound.argtypes = [c_vp, c_i64, c_i64, c_dbl, c_vp, c_sz, c_vp, ctypes.POINTER(c_dbl)]
    lib.ns_shift_certificate.restype = ctypes.c_int
    lib.ns_shift_certificate.argtypes = [c_dbl, c_dbl, c_dbl, c_dbl, c_dbl, ctypes.POINTER(NsShiftCert)]
    lib.ns_workspace_bytes_alg1.restype = c_sz
    lib.ns_workspace_bytes_alg1.argtypes = [c_i32]
    lib.ns_alg1_rotated_quartic.restype = ctypes.c_int
    lib.ns_alg1_rotated_quartic.argtypes = [c_vp, c_i64, c_i32, c_vp, c_vp, c_i32, c_dbl, c_i32, c_dbl, c_vp, c_vp,
                                            c_sz, c_vp, ctypes.POINTER(NsAlg1Result)]
    lib.ns_alg1_rotated_quartic_ex.restype = ctypes.c_int
    lib.ns_alg1_rotated_quartic_ex.argtypes = [c_vp, c_i64, c_i32, c_vp, c_vp, c_i32, c_dbl, c_i32, c_dbl,
                                               ctypes.POINTER(NsAlg1Policy), c_vp, c_vp, c_sz, c_vp,
                                               ctypes.POINTER(NsAlg1Result)]
    _lib = lib
    return lib


def _check(st):
    if st != NS_OK:
        lib = load_library()
        raise NsError(f"{lib.ns_status_string(st).decode()}: {lib.ns_last_error().decode()}")


_TORCH = None
_RAW_STREAM = None


def _torch():
    global _TORCH
    if _TORCH is None:      # imported lazily (the package itself does not need torch), then cached:
        import torch        # this sits on the small-d latency path, several calls per reflector
        _TORCH = torch
    return _TORCH


def _stream_ptr(stream, device=None):
    """cudaStream_t of `stream`, or of torch's current stream on `device` (the raw-handle query avoids
    building a torch.cuda.Stream object: ~3 us per call on the small-d latency path)."""
    global _RAW_STREAM
    torch = _torch()
    if stream is not None:
        return ctypes.c_void_p(stream.cuda_stream)
    if _RAW_STREAM is None:
        _RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", False)
    raw = _RAW_STREAM
    if raw:
        idx = device.index if device is not None and device.index is not None else torch.cuda.current_device()
        return ctypes.c_void_p(raw(idx))
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


class _NullCtx:
    def __enter__(self):
        return None

    def __exit__(self, *a):
        return False


_NULL = _NullCtx()


def _on(dev):
    """Make `dev` the current CUDA device for one C call: the library launches on the current device and
    queries no tensor's device itself.  A no-op (no torch context object) when it already is current, which
    keeps the small-d latency path free of the device switch."""
    torch = _torch()
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    if idx == torch.cuda.current_device():
        return _NULL
    return torch.cuda.device(idx)


def _require_cuda_f64(t, name):
    torch = _torch()
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64):
        raise NsError(f"{name} must be a CUDA float64 tensor (no CPU fallback)")


def _same_device(*ts):
    dev = ts[0].device
    for t in ts[1:]:
        if t.device != dev:
            raise NsError(f"all tensors of one call must be on the same device ({dev} vs {t.device})")


def ns_workspace_bytes(d, prec=NS_PREC_FP64):
    return load_library().ns_workspace_bytes(d, prec)


def ns_workspace_bytes_batched(d, batch, prec=NS_PREC_FP64):
    return load_library().ns_workspace_bytes_batched(d, batch, prec)


def alloc_workspace(nbytes, device):
    torch = _torch()
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device)


def ns_options(**kw):
    """ns_options_t with library defaults, fields overridden by keyword (switch_tol, cg_iters, ...)."""
    o = NsOptions()
    load_library().ns_options_default(ctypes.byref(o))
    for k_, v in kw.items():
        if k_ == "filter_c":
            v = (ctypes.c_double * 3)(*(list(v) + [0.0] * (3 - len(v))))
        setattr(o, k_, v)
    return o


def ns_reflector(H, s, alpha, k, max_steps, tol, tol_mode=NS_TOL_ABS, prec=NS_PREC_FP64, R=None, ws=None,
                 stream=None, options=None):
    """R = sgn(H - sI) by Newton–Schulz on the GPU (C-ABI ns_reflector / ns_reflector_ex when options
    are given).  Returns (R, result dict).  (Written for the small-d latency path: device checks on integer
    indices, the raw stream handle, no context object unless a device switch is needed.)"""
    torch = _torch()
    lib = _lib if _lib is not None else load_library()
    dev = H.get_device() if isinstance(H, torch.Tensor) else -1
    if dev < 0 or H.dtype != torch.float64:
        raise NsError("H must be a CUDA float64 tensor (no CPU fallback)")
    d = H.shape[0]
    if H.dim() != 2 or H.shape[1] != d or H.stride(1) != 1:
        raise NsError("H must be a square row-major (stride(1)==1) matrix")
    if R is None:
        R = torch.empty((d, d), dtype=torch.float64, device=H.device)
    elif not isinstance(R, torch.Tensor) or R.get_device() != dev or R.dtype != torch.float64:
        raise NsError("R must be a CUDA float64 tensor on H's device")
    if ws is None:   # (the library checks a given size)
        nb = lib.ns_workspace_bytes_ex(d, prec, ctypes.byref(options)) if options is not None else \
            lib.ns_workspace_bytes(d, prec)
        ws = alloc_workspace(nb, H.device)
    elif ws.get_device() != dev:
        raise NsError("the workspace must be on H's device")
    res = NsResult()
    if stream is not None:
        sp = ctypes.c_void_p(stream.cuda_stream)
    else:
        sp = _stream_ptr(None, H.device)
    args = (ctypes.c_void_p(H.data_ptr()), d, H.stride(0), float(s), float(alpha), int(k), int(max_steps), float(tol),
            int(tol_mode), int(prec), ctypes.c_void_p(R.data_ptr()), R.stride(0), ctypes.c_void_p(ws.data_ptr()),
            ws.numel(), sp)
    with (_NULL if dev == torch._C._cuda_getDevice() else torch.cuda.device(dev)):
        if options is None:
            st = lib.ns_reflector(*args, ctypes.byref(res))
        else:
            st = lib.ns_reflector_ex(*args, ctypes.byref(options), ctypes.byref(res))
    if st != NS_OK:
        _check(st)
    return R, res.as_dict()


def ns_reflector_host(H, s, alpha, k, max_steps, tol, tol_mode=NS_TOL_ABS, prec=NS_PREC_FP64, R=None, ws=None,
                      stream=None, device=None):
    """End-to-end entry: host (numpy or pinned CPU torch) H in, host R out (C-ABI ns_reflector_host)."""
    torch = _torch()
    lib = load_library()
    if isinstance(H, np.ndarray):
        H = torch.from_numpy(np.ascontiguousarray(H, dtype=np.float64))
    if H.is_cuda or H.dtype != torch.float64:
        raise NsError("H must be a CPU float64 tensor/array")
    d = H.shape[0]
    if R is None:
        R = torch.empty((d, d), dtype=torch.float64, pin_memory=H.is_pinned())
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else device
    if ws is None:
        ws = alloc_workspace(lib.ns_workspace_bytes_host(d, prec), dev)
    if ws.device.type != "cuda":
        raise NsError("the workspace must be device memory")
    dev = ws.device
    res = NsResult()
    with _on(dev):
        st = lib.ns_reflector_host(ctypes.c_void_p(H.data_ptr()), d, H.stride(0), float(s), float(alpha), int(k),
                                   int(max_steps), float(tol), int(tol_mode), int(prec), ctypes.c_void_p(R.data_ptr()),
                                   R.stride(0), ctypes.c_void_p(ws.data_ptr()), ws.numel(), _stream_ptr(stream, dev),
                                   ctypes.byref(res))
    _check(st)
    return R, res.as_dict()


def ns_reflector_batched(H, s, alpha, k, max_steps, tol, tol_mode=NS_TOL_ABS, prec=NS_PREC_FP64, R=None, ws=None,
                         stream=None):
    """Batched reflectors: H (batch, d, d) CUDA float64; s, alpha, k per problem (host sequences)."""
    torch = _torch()
    lib = load_library()
    _require_cuda_f64(H, "H")
    if H.dim() != 3 or H.shape[1] != H.shape[2] or not H.is_contiguous():
        raise NsError("H must be a contiguous (batch, d, d) tensor")
    b, d = H.shape[0], H.shape[1]
    s_a = np.ascontiguousarray(np.broadcast_to(np.asarray(s, dtype=np.float64), (b,)))
    a_a = np.ascontiguousarray(np.broadcast_to(np.asarray(alpha, dtype=np.float64), (b,)))
    k_a = np.ascontiguousarray(np.broadcast_to(np.asarray(k, dtype=np.int32), (b,)))
    if R is None:
        R = torch.empty_like(H)
    _require_cuda_f64(R, "R")
    if ws is None:
        ws = alloc_workspace(lib.ns_workspace_bytes_batched(d, b, prec), H.device)
    if R.shape != H.shape or not R.is_contiguous():
        raise NsError("R must be a contiguous tensor of H's shape")
    _same_device(H, R, ws)
    outs = (NsResult * b)()
    with _on(H.device):
        st = lib.ns_reflector_batched(ctypes.c_void_p(H.data_ptr()), d, b, H.stride(0), s_a.ctypes.data,
                                      a_a.ctypes.data, k_a.ctypes.data, int(max_steps), float(tol), int(tol_mode),
                                      int(prec), ctypes.c_void_p(R.data_ptr()), R.stride(0),
                                      ctypes.c_void_p(ws.data_ptr()), ws.numel(), _stream_ptr(stream, H.device), outs)
    _check(st)
    return R, _ResultList(outs)


def ns_reflector_batched_dev(H, s, alpha, k, max_steps, tol, tol_mode=NS_TOL_ABS, prec=NS_PREC_FP64, R=None,
                             ws=None, stream=None):
    """Batched reflectors with the per-problem s, alpha, k as CUDA tensors (float64, float64, int32)."""
    torch = _torch()
    lib = load_library()
    _require_cuda_f64(H, "H")
    if H.dim() != 3 or H.shape[1] != H.shape[2] or not H.is_contiguous():
        raise NsError("H must be a contiguous (batch, d, d) tensor")
    b, d = H.shape[0], H.shape[1]
    for name, t, dt in (("s", s, torch.float64), ("alpha", alpha, torch.float64), ("k", k, torch.int32)):
        if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == dt and t.numel() == b and t.is_contiguous()):
            raise NsError(f"{name} must be a contiguous CUDA {dt} tensor of {b} elements")
    if R is None:
        R = torch.empty_like(H)
    if ws is None:
        ws = alloc_workspace(lib.ns_workspace_bytes_batched(d, b, prec), H.device)
    _same_device(H, R, ws, s, alpha, k)
    outs = (NsResult * b)()
    with _on(H.device):
        st = lib.ns_reflector_batched_dev(ctypes.c_void_p(H.data_ptr()), d, b, H.stride(0), ctypes.c_void_p(s.data_ptr()),
                                          ctypes.c_void_p(alpha.data_ptr()), ctypes.c_void_p(k.data_ptr()),
                                          int(max_steps), float(tol), int(tol_mode), int(prec),
                                          ctypes.c_void_p(R.data_ptr()), R.stride(0), ctypes.c_void_p(ws.data_ptr()),
                                          ws.numel(), _stream_ptr(stream, H.device), outs)
    _check(st)
    return R, _ResultList(outs)


def ns_inertia(H, s, prec=NS_PREC_FP64, max_steps=100, ws=None, stream=None):
    """#{lambda_i(H) < s} from the Newton–Schulz trace certificate (C-ABI ns_inertia).
    Returns (count, resolved, result dict)."""
    lib = load_library()
    _require_cuda_f64(H, "H")
    d = H.shape[0]
    if H.dim() != 2 or H.shape[1] != d or H.stride(1) != 1:
        raise NsError("H must be a square row-major matrix")
    if ws is None:
        ws = alloc_workspace(lib.ns_workspace_bytes_inertia(d, prec), H.device)
    c, r, res = ctypes.c_int64(), ctypes.c_int32(), NsResult()
    with _on(H.device):
        st = lib.ns_inertia(ctypes.c_void_p(H.data_ptr()), d, H.stride(0), float(s), int(prec), int(max_steps),
                            ctypes.c_void_p(ws.data_ptr()), ws.numel(), _stream_ptr(stream, H.device), ctypes.byref(c),
                            ctypes.byref(r), ctypes.byref(res))
    _check(st)
    return c.value, bool(r.value), res.as_dict()


def ns_shift_bisect(H, k, lo=0.0, hi=0.0, rel_eps=0.05, max_probes=200, prec=NS_PREC_FP64, ws=None, stream=None):
    """Certified midpoint shift for the gap (lambda_k, lambda_k+1) by inertia-probe bisection (C-ABI
    ns_shift_bisect).  lo >= hi: default bracket [-||H||_inf, ||H||_inf].  Returns a dict."""
    lib = load_library()
    _require_cuda_f64(H, "H")
    d = H.shape[0]
    if H.dim() != 2 or H.shape[1] != d or H.stride(1) != 1:
        raise NsError("H must be a square row-major matrix")
    if ws is None:
        ws = alloc_workspace(lib.ns_workspace_bytes_inertia(d, prec), H.device)
    o = NsBisect()
    with _on(H.device):
        st = lib.ns_shift_bisect(ctypes.c_void_p(H.data_ptr()), d, H.stride(0), int(k), float(lo), float(hi),
                                 float(rel_eps), int(max_probes), int(prec), ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                 _stream_ptr(stream, H.device), ctypes.byref(o))
    _check(st)
    return {f: getattr(o, f) for f, _ in NsBisect._fields_ if f != "pad"}


def ns_symm_product(A, B, mode=0, C=None, ws=None, stream=None, prec=NS_PREC_FP64):
    """C = A B (mode 0, symmetric tiles), 1.5 A - 0.5 A B (mode 1) or A B on every tile (mode 2);
    A, B symmetric (upper triangles read).  prec selects the FP64 DMMA or BF16x3 tcgen05 core."""
    torch = _torch()
    lib = load_library()
    _require_cuda_f64(A, "A")
    _require_cuda_f64(B, "B")
    d = A.shape[0]
    for name, t in (("A", A), ("B", B)):
        if t.dim() != 2 or tuple(t.shape) != (d, d) or t.stride(1) != 1:
            raise NsError(f"{name} must be a (d, d) row-major (stride(1) == 1) matrix")
    if A.stride(0) != B.stride(0):
        raise NsError("A and B must share a leading dimension")
    ld = A.stride(0)
    if C is None:
        # the library writes C with A's leading dimension: allocate exactly that layout (rows of ld doubles;
        # torch.empty_strided sizes the storage for the last row's d elements, not a full pitch)
        C = torch.empty_strided((d, d), (ld, 1), dtype=torch.float64, device=A.device)
    _require_cuda_f64(C, "C")
    if C.dim() != 2 or tuple(C.shape) != (d, d) or C.stride(1) != 1 or C.stride(0) != ld:
        raise NsError("C must be a (d, d) row-major matrix with A's leading dimension")
    if ws is None:
        ws = alloc_workspace(lib.ns_workspace_bytes(d, prec), A.device)
    _same_device(A, B, C, ws)
    with _on(A.device):
        st = lib.ns_symm_product(ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()),
                                 ctypes.c_void_p(C.data_ptr()), d, ld, int(mode), int(prec),
                                 ctypes.c_void_p(ws.data_ptr()), ws.numel(), _stream_ptr(stream, A.device))
    _check(st)
    return C



def ns_reflector_sharded_emulated(nranks, H, s, alpha, k, max_steps, tol, tol_mode=NS_TOL_ABS, R=None, ws=None,
                                  stream=None, rows=False, sender_mirror=False):
    """The sharded algorithm with `nranks` ranks emulated on one GPU (C-ABI ns_reflector_sharded_emulated)."""
    torch = _torch()
    lib = load_library()
    _require_cuda_f64(H, "H")
    d = H.shape[0]
    if R is None:
        R = torch.empty((d, d), dtype=torch.float64, device=H.device)
    if ws is None:
        ws = alloc_workspace(lib.ns_workspace_bytes_sharded_emulated(d, nranks), H.device)
    res = NsResult()
    with _on(H.device):
        st = lib.ns_reflector_sharded_emulated(int(nranks), ctypes.c_void_p(H.data_ptr()), d, H.stride(0), float(s),
                                           float(alpha), int(k), int(max_steps), float(tol), int(tol_mode),
                                           ctypes.c_void_p(R.data_ptr()), R.stride(0), ctypes.c_void_p(ws.data_ptr()),
                                           ws.numel(), _stream_ptr(stream, H.device),
                                           (1 if rows else 0) | (2 if sender_mirror else 0), ctypes.byref(res))
    _check(st)
    return R, res.as_dict()


def ns_symm_product_shard(A, B, C_list, rank, nranks, mode=0, ws=None, stream=None):
    """Peer-memory exchange primitive (C-ABI ns_symm_product_shard): rank `rank`'s tiles of the
    symmetric product, each stored into every matrix of C_list (CUDA float64, d x d, d % 128 == 0)."""
    lib = load_library()
    _require_cuda_f64(A, "A")
    _require_cuda_f64(B, "B")
    d = A.shape[0]
    for C in C_list:
        _require_cuda_f64(C, "C")
    if ws is None:
        ws = alloc_workspace(lib.ns_workspace_bytes(d, NS_PREC_FP64), A.device)
    arr = (ctypes.c_void_p * len(C_list))(*[C.data_ptr() for C in C_list])
    with _on(A.device):
        st = lib.ns_symm_product_shard(ctypes.c_void_p(A.data_ptr()), ctypes.c_void_p(B.data_ptr()), arr, len(C_list), d,
                                   int(mode), int(rank), int(nranks), ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                   _stream_ptr(stream, A.device))
    _check(st)


def ns_profile_enable(on=True):
    load_library().ns_profile_enable(1 if on else 0)


def ns_profile_reset():
    load_library().ns_profile_reset()


def ns_profile_get():
    p = NsProfile()
    load_library().ns_profile_get(ctypes.byref(p))
    return {f: getattr(p, f) for f, _ in NsProfile._fields_}


def ns_comm_get_unique_id():
    """128-byte NCCL unique id (rank 0 creates it; broadcast it to the other ranks)."""
    buf = ctypes.create_string_buffer(128)
    _check(load_library().ns_comm_get_unique_id(buf))
    return buf.raw


def ns_comm_init(rank, nranks, uid):
    """NCCL communicator for the sharded path (collective across ranks; current CUDA device)."""
    h = ctypes.c_void_p()
    _check(load_library().ns_comm_init(int(rank), int(nranks), bytes(uid), ctypes.byref(h)))
    return h


def ns_comm_init_host(rank, nranks, allgather):
    """Communicator without NCCL (C-ABI ns_comm_init_host): `allgather(data: bytes) -> list[bytes]` must
    all-gather one bytes object per rank (e.g. over a gloo process group).  Lets several processes share one
    GPU in tests: the library's barriers become stream syncs + this host exchange."""
    def _cb(send, recv, nbytes, user):
        try:
            parts = allgather(ctypes.string_at(send, nbytes))
            buf = b"".join(parts)
            if len(buf) != nbytes * nranks:
                raise NsError(f"host all-gather returned {len(buf)} bytes, expected {nbytes} x {nranks}")
            ctypes.memmove(recv, buf, len(buf))
            return 0
        except Exception:      # noqa: BLE001 -- an exception must not cross the C frame
            import sys
            import traceback
            traceback.print_exc(file=sys.stderr)
            return 1
    fn = HOST_ALLGATHER(_cb)
    h = ctypes.c_void_p()
    _check(load_library().ns_comm_init_host(int(rank), int(nranks), fn, None, ctypes.byref(h)))
    _HOST_CALLBACKS[h.value] = fn
    return h


def ns_comm_destroy(comm):
    _check(load_library().ns_comm_destroy(comm))
    _HOST_CALLBACKS.pop(getattr(comm, "value", None), None)


def ns_shard_rows(d, nranks, rank):
    """[row0, row1) of the block-row panel rank `rank` owns in the rows entry (host-only)."""
    a, b = ctypes.c_int64(), ctypes.c_int64()
    _check(load_library().ns_shard_rows(int(d), int(nranks), int(rank), ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def ns_shard_plan(d, nranks, rank):
    """(n, 2) int32 array of the (I, J) upper tiles rank `rank` computes (host-only)."""
    lib = load_library()
    n = ctypes.c_int32()
    _check(lib.ns_shard_plan(int(d), int(nranks), int(rank), None, 0, ctypes.byref(n)))
    out = np.zeros((max(n.value, 1), 2), dtype=np.int32)
    _check(lib.ns_shard_plan(int(d), int(nranks), int(rank), out.ctypes.data, n.value, ctypes.byref(n)))
    return out[:n.value]


def ns_shard_chunks(d, nranks):
    """(n_chunks, chunk_slots) of the sharded exchange (host-only)."""
    a, b = ctypes.c_int32(), ctypes.c_int32()
    _check(load_library().ns_shard_chunks(int(d), int(nranks), ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def ns_workspace_bytes_sharded(d, nranks):
    return load_library().ns_workspace_bytes_sharded(d, nranks)


def ns_reflector_sharded(comm, H, s, alpha, k, max_steps, tol, tol_mode=NS_TOL_ABS, R=None, ws=None, stream=None,
                         nranks=None):
    """Multi-GPU reflector (every rank passes the full H; every rank receives the full R)."""
    torch = _torch()
    lib = load_library()
    _require_cuda_f64(H, "H")
    d = H.shape[0]
    if R is None:
        R = torch.empty((d, d), dtype=torch.float64, device=H.device)
    if ws is None:
        ws = alloc_workspace(lib.ns_workspace_bytes_sharded(d, nranks or 1), H.device)
    res = NsResult()
    with _on(H.device):
        st = lib.ns_reflector_sharded(comm, ctypes.c_void_p(H.data_ptr()), d, H.stride(0), float(s), float(alpha), int(k),
                                  int(max_steps), float(tol), int(tol_mode), ctypes.c_void_p(R.data_ptr()), R.stride(0),
                                  ctypes.c_void_p(ws.data_ptr()), ws.numel(), _stream_ptr(stream, H.device),
                                  ctypes.byref(res))
    _check(st)
    return R, res.as_dict()


def ns_reflector_sharded_rows(comm, H_rows, d, s, alpha, k, max_steps, tol, tol_mode=NS_TOL_ABS, R_rows=None,
                              ws=None, stream=None, nranks=None, prec=NS_PREC_FP64):
    """Multi-GPU reflector on block-row panels (C-ABI ns_reflector_sharded_rows): H_rows = this rank's rows
    [row0, row1) of H ((d/P, d) CUDA float64, stride(1) == 1); returns (R_rows, result)."""
    torch = _torch()
    lib = load_library()
    _require_cuda_f64(H_rows, "H_rows")
    if H_rows.dim() != 2 or H_rows.shape[1] != d or H_rows.stride(1) != 1:
        raise NsError("H_rows must be a (rows, d) row-major matrix")
    if R_rows is None:
        R_rows = torch.empty(tuple(H_rows.shape), dtype=torch.float64, device=H_rows.device)
    _require_cuda_f64(R_rows, "R_rows")
    if tuple(R_rows.shape) != tuple(H_rows.shape) or R_rows.stride(1) != 1:
        raise NsError("R_rows must have H_rows' shape, row-major")
    if ws is None:
        ws = alloc_workspace(lib.ns_workspace_bytes_sharded(d, nranks or 1), H_rows.device)
    _same_device(H_rows, R_rows, ws)
    res = NsResult()
    with _on(H_rows.device):
        st = lib.ns_reflector_sharded_rows(comm, ctypes.c_void_p(H_rows.data_ptr()), int(d), H_rows.stride(0),
                                           float(s), float(alpha), int(k), int(max_steps), float(tol), int(tol_mode),
                                           int(prec), ctypes.c_void_p(R_rows.data_ptr()), R_rows.stride(0),
                                           ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                           _stream_ptr(stream, H_rows.device), ctypes.byref(res))
    _check(st)
    return R_rows, res.as_dict()


def ns_scale_bound(H, s, ws=None, stream=None):
    """||H - sI||_inf on the device (Gershgorin alpha; upper triangle read)."""
    lib = load_library()
    _require_cuda_f64(H, "H")
    d = H.shape[0]
    if ws is None:
        ws = alloc_workspace(lib.ns_workspace_bytes_setup(d), H.device)
    out = ctypes.c_double()
    with _on(H.device):
        st = lib.ns_scale_bound(ctypes.c_void_p(H.data_ptr()), d, H.stride(0), float(s), ctypes.c_void_p(ws.data_ptr()),
                                ws.numel(), _stream_ptr(stream, H.device), ctypes.byref(out))
    _check(st)
    return out.value


def ns_shift_certificate(lam_k_hat, lam_k1_hat, eps, s, delta=0.0):
    """prop:reuse_refresh certificate (host-only C function)."""
    c = NsShiftCert()
    _check(load_library().ns_shift_certificate(float(lam_k_hat), float(lam_k1_hat), float(eps), float(s),
                                               float(delta), ctypes.byref(c)))
    return dict(margin_hat=c.margin_hat, margin_lb=c.margin_lb, reuse_margin_lb=c.reuse_margin_lb,
                midpoint=c.midpoint, admissible=bool(c.admissible), reuse_ok=bool(c.reuse_ok),
                midpoint_ok=bool(c.midpoint_ok))


def ns_alg1_rotated_quartic(Q, k, x0, m, eta, max_iters, grad_tol, x_out=None, ws=None, stream=None,
                            policy="midpoint", damp=0.5, clip=0.25, reuse_margin=0.0, eps=0.0):
    """Batched Algorithm 1 on the rotated quartic (N2).  Q (d, d) and x0 (nruns, d) CUDA float64;
    k host ints; policy "midpoint" | "damped" | "reuse_refresh" with its parameters and the admissibility
    bound eps (ns_alg1_rotated_quartic_ex).  Returns (x_final, list of result dicts)."""
    torch = _torch()
    lib = load_library()
    _require_cuda_f64(Q, "Q")
    _require_cuda_f64(x0, "x0")
    nruns, d = x0.shape
    k_a = np.ascontiguousarray(np.broadcast_to(np.asarray(k, dtype=np.int32), (nruns,)))
    if x_out is None:
        x_out = torch.empty_like(x0)
    if ws is None:
        ws = alloc_workspace(lib.ns_workspace_bytes_alg1(nruns), x0.device)
    if policy not in NS_SHIFT_POLICIES:
        raise ValueError(f"unknown shift policy {policy!r}")
    pol = NsAlg1Policy(NS_SHIFT_POLICIES[policy], 0, float(damp), float(clip), float(reuse_margin), float(eps))
    outs = (NsAlg1Result * nruns)()
    with _on(x0.device):
        st = lib.ns_alg1_rotated_quartic_ex(ctypes.c_void_p(Q.data_ptr()), d, nruns, k_a.ctypes.data,
                                            ctypes.c_void_p(x0.data_ptr()), int(m), float(eta), int(max_iters),
                                            float(grad_tol), ctypes.byref(pol), ctypes.c_void_p(x_out.data_ptr()),
                                            ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                            _stream_ptr(stream, x0.device), outs)
    _check(st)
    return x_out, [dict(iters=o.iters, morse_index=o.morse_index, success=bool(o.success), grad_norm=o.grad_norm,
                        stop_reason=o.stop_reason, refreshes=o.refreshes, s_last=o.s_last) for o in outs]


def build_info():
    return load_library().ns_build_info().decode()
