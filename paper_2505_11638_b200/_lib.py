"""ctypes binding of libngd_b200.so (include/ngd.h) and the device-array helpers.

There is no CPU fallback: if the shared library is missing or no CUDA device is
visible, every compute entry point raises.  Device arrays are torch CUDA
tensors (PyTorch is the allocator/stream plumbing); all arithmetic runs in the
library's sm_100a kernels, cuBLAS/cuSOLVER calls and NCCL collectives.
"""

from __future__ import annotations

import contextlib
import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libngd_b200.so")
LIB_PATH = os.environ.get("NGD_LIB_PATH", LIB_PATH)  # tuning experiments: an alternative build of the library

NGD_OK, NGD_E_SHAPE, NGD_E_NONFINITE, NGD_E_CHOL, NGD_E_CUDA, NGD_E_NCCL, NGD_E_STATE = range(7)


class NonFiniteError(ArithmeticError):
    """A computation produced a NaN or Inf value (autodiff.py:48-49)."""


class CholeskyFailure(RuntimeError):
    """Omega^T Y_nu was not numerically positive definite (sketch.py:76-78)."""


class SolveReportC(ctypes.Structure):
    _fields_ = [
        ("iterations", ctypes.c_int32),
        ("matvecs", ctypes.c_int32),
        ("converged", ctypes.c_int32),
        ("breakdown", ctypes.c_int32),
        ("relative_residual", ctypes.c_double),
    ]


_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_I32 = ctypes.c_int32
_D = ctypes.c_double

# name -> argtypes (all functions return int status unless listed in _RESTYPE)
SIGNATURES = {
    "ngd_last_error": [],
    "ngd_version": [],
    "ngd_ctx_create": [ctypes.POINTER(_I32), _I32, _I32, ctypes.POINTER(_P)],
    "ngd_ctx_destroy": [_P],
    "ngd_ctx_set_stream": [_P, _P],
    "ngd_param_count": [_P],
    "ngd_nccl_unique_id": [ctypes.c_char_p],
    "ngd_ctx_set_comm": [_P, ctypes.c_char_p, _I32, _I32],
    "ngd_set_points": [_P, _I64, _P, _P, _P, _I64, _P, _P, _P],
    "ngd_set_rows": [_P, _I64, _P, _P, _P, _P, _I64, _P, _P, _P, _P],
    "ngd_set_head": [_P, _P, _I32, _D, ctypes.c_uint32],
    "ngd_loss": [_P, _P, ctypes.POINTER(_D)],
    "ngd_loss_at": [_P, _P, _D, _P, ctypes.POINTER(_D)],
    "ngd_linearize": [_P, _P, ctypes.POINTER(_D), _P],
    "ngd_gram_dense": [_P, _P, _I64],
    "ngd_small_cholesky": [_P, _P, _I32, _I32, ctypes.POINTER(_I32)],
    "ngd_h1_error": [_P, _P, _P, ctypes.POINTER(_D)],
    "ngd_linearize_ex": [_P, _P, _P, ctypes.POINTER(_D), _P, _P],
    "ngd_loss_grad": [_P, _P],
    "ngd_jvp": [_P, _P, _P],
    "ngd_vjp": [_P, _P, _P],
    "ngd_gram_matvec": [_P, _P, _D, _P],
    "ngd_gram_matmat": [_P, _P, _I64, _I64, _P, _I64],
    "ngd_fill_gaussian": [_P, ctypes.c_uint64, _P, _I64],
    "ngd_nystrom_prepare": [_P, _P, _I64, _I32],
    "ngd_nystrom_finish": [_P, _P, _P, _I64, _I32, _P, _P, ctypes.POINTER(_D)],
    "ngd_dense_matmat": [_P, _P, _I64, _P, _I64, _P],
    "ngd_gemm": [_P, _I32, _I32, _I32, _I32, _I32, _D, _P, _I64, _P, _I64, _D, _P, _I64],
    "ngd_gemm_ozaki": [_P, _I32, _I32, _I32, _D, _P, _I64, _P, _I64, _D, _P, _I64],
    "ngd_precond_apply": [_P, _P, _P, _I32, _D, _P, _P, _I64],
    "ngd_pcg": [_P, _P, _I64, _P, _D, _P, _P, _I32, _D, _D, _I32, _I32, _P, ctypes.POINTER(SolveReportC)],
    "ngd_small_svd": [_P, _P, _I32, _P, _P, _I32, ctypes.POINTER(_I32)],
    "ngd_get_stat": [_P, ctypes.c_char_p, ctypes.POINTER(_I64)],
    "ngd_set_option": [_P, ctypes.c_char_p, _I64],
    "ngd_dot": [_P, _P, _P, _I64, ctypes.POINTER(_D)],
    "ngd_axpy": [_P, _P, _D, _P, _P, _I64],
    "ngd_stream_sync": [_P],
    "ngd_launch_count": [],
    "ngd_gemm_flops": [],
    "ngd_i8_ops": [],
    "ngd_oz_conv_elems": [],
    "ngd_phase_flops": [_I32],
    "ngd_probe_start": [_I32, _I32],
    "ngd_probe_stop": [ctypes.POINTER(_D), ctypes.POINTER(_I64)],
    "ngd_probe_stop_all": [ctypes.POINTER(_D), ctypes.POINTER(_I64), _I32],
}
_RESTYPE = {"ngd_last_error": ctypes.c_char_p, "ngd_param_count": _I64, "ngd_launch_count": _I64,
            "ngd_gemm_flops": _D, "ngd_i8_ops": _D, "ngd_oz_conv_elems": _D, "ngd_phase_flops": _D}

_lib = None
_contexts = []  # weak registry so option changes reach live contexts
OPTIONS = {"svd": 3}


# library defaults of the ngd_set_option knobs (include/ngd.h), for restoring a temporary change
DEFAULTS = {"svd": 3, "graphs": 1, "l2window": 1, "force_comm": 0, "pdl": 1, "l2u": 1, "sketch_gemm": 2, "i8_pair": 1,
            "pha_gemm": 2, "out_pre": 2, "oz_max_blocks": 1024}


@contextlib.contextmanager
def option(key, value):
    """Temporarily set a library knob (restores the previous or default value on exit)."""
    prev = OPTIONS.get(key, DEFAULTS.get(key))
    set_option(key, value)
    try:
        yield
    finally:
        if prev is None:
            OPTIONS.pop(key, None)
        else:
            set_option(key, prev)


def set_option(key, value):
    """Set a library knob on every live and future context (see ngd_set_option).  A value the
    library rejects raises (ValueError) and leaves the process-wide setting unchanged."""
    live = [c for c in (r() for r in list(_contexts)) if c is not None and c._h is not None]
    if live:
        live[0].call("ngd_set_option", key.encode(), int(value))  # validates first
    OPTIONS[key] = int(value)
    for ctx in live[1:]:
        ctx.call("ngd_set_option", key.encode(), int(value))


def load():
    """Load the shared library (raises if it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} not found: build it with `python -m paper_2505_11638_b200.build` "
            "(there is no CPU fallback)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, args in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = _RESTYPE.get(name, ctypes.c_int)
    _lib = lib
    return lib


def check(rc):
    if rc == NGD_OK:
        return
    msg = load().ngd_last_error().decode(errors="replace")
    if rc == NGD_E_SHAPE:
        raise ValueError(msg)
    if rc == NGD_E_NONFINITE:
        raise NonFiniteError(msg)
    if rc == NGD_E_CHOL:
        raise CholeskyFailure(msg)
    raise RuntimeError(f"libngd_b200 error {rc}: {msg}")


# ---------------------------------------------------------------------------
# device arrays
# ---------------------------------------------------------------------------


def torch_mod():
    import torch

    return torch


def device():
    torch = torch_mod()
    if not torch.cuda.is_available():
        raise RuntimeError("no CUDA device visible: the B200 path has no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def is_device_array(x):
    torch = torch_mod()
    return isinstance(x, torch.Tensor) and x.is_cuda


def to_device(x, dtype=None):
    """numpy/list/torch -> contiguous float64 CUDA tensor (no copy if already one)."""
    torch = torch_mod()
    if isinstance(x, torch.Tensor):
        t = x
        if not t.is_cuda:
            t = t.to(device())
        if t.dtype != torch.float64:
            t = t.to(torch.float64)
        return t.contiguous()
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    return torch.from_numpy(arr).to(device(), non_blocking=False)


def like_input(t, ref):
    """Return t (a CUDA tensor) in the array namespace of ``ref`` (numpy in -> numpy out)."""
    if is_device_array(ref):
        return t
    return t.detach().cpu().numpy()


def ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


class Context:
    """One libngd context (topology + device workspace) on the current CUDA device."""

    def __init__(self, widths):
        torch = torch_mod()
        lib = load()
        dev = device()
        w = (_I32 * len(widths))(*[int(x) for x in widths])
        h = _P()
        check(lib.ngd_ctx_create(w, len(widths), dev.index, ctypes.byref(h)))
        self._h = h
        self.lib = lib
        self.widths = tuple(int(x) for x in widths)
        self.device = dev
        self.stream = torch.cuda.current_stream(dev)
        check(lib.ngd_ctx_set_stream(h, _P(self.stream.cuda_stream)))
        self.p = int(lib.ngd_param_count(h))
        self.points_key = None
        self.lin_token = 0
        self.lin_owner = None
        import weakref

        for k, v in OPTIONS.items():
            self.call("ngd_set_option", k.encode(), int(v))
        _contexts.append(weakref.ref(self))

    @property
    def handle(self):
        return self._h

    def call(self, name, *args):
        check(getattr(self.lib, name)(self._h, *args))

    def close(self):
        if getattr(self, "_h", None) is not None and self.lib is not None:
            self.lib.ngd_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
