"""GPU real-FFT backend: drop-in for the reference's pluggable
``stagflow.transforms.rfftn / irfftn`` (transforms.py:9-12; looked up by the
spectral solver at poisson.py:196,199; contract pinned by
test_poisson.py:273-283: round trip within 4 ulp, dtype preserved).

Transforms run over every axis of a 1-3 dimensional array.  CUDA tensors stay
on the device; numpy arrays are copied in and the result copied back, so code
written against scipy's signature keeps working.  2/3/5/7-smooth shapes with
an even last axis use the hand-written engine; others use cuFFT
(``uses_own_engine`` tells which).  The GPU spectral solver does not go
through these functions: its transforms are fused with the divergence and the
eigenvalue scaling (csrc/fft.cu)."""

import ctypes

import numpy as np
import torch

from . import _native as N
from .plan import stream_ptr

_PLANS = {}
_CPLX = {torch.float64: torch.complex128, torch.float32: torch.complex64}
_REAL = {torch.complex128: torch.float64, torch.complex64: torch.float32}


class _Plan:
    def __init__(self, shape, dtype):
        n = (ctypes.c_int * 3)(*(list(shape) + [1] * (3 - len(shape))))
        h = N.vp()
        N.check(N.lib.sfb_fft_create(len(shape), n, 0 if dtype == torch.float64 else 1, ctypes.byref(h)))
        self.handle = h.value
        self.own = bool(N.lib.sfb_fft_uses_own(self.handle))
        # hand-written launches per transform: R2C/C2R + one pass per other axis
        N._FFT_PASSES[self.handle] = len(shape) if self.own else 0

    def __del__(self):
        try:
            N._FFT_PASSES.pop(self.handle, None)
            N.lib.sfb_fft_destroy(self.handle)
        except Exception:  # noqa: BLE001 - interpreter shutdown
            pass


def _plan(shape, dtype):
    key = (tuple(int(v) for v in shape), dtype)
    p = _PLANS.get(key)
    if p is None:
        p = _PLANS[key] = _Plan(key[0], dtype)
    return p


def _check_axes(x, s, axes):
    if axes is not None and tuple(axes) != tuple(range(x.ndim)):
        raise ValueError("only transforms over all axes are supported (the reference's usage)")
    if not 1 <= x.ndim <= 3:
        raise ValueError("rfftn/irfftn support 1-3 dimensions")


def _to_device(x, dtypes):
    host = not isinstance(x, torch.Tensor)
    t = torch.from_numpy(np.ascontiguousarray(x)) if host else x
    if t.dtype not in dtypes:
        raise TypeError(f"unsupported dtype {t.dtype}")
    return t.to("cuda", non_blocking=False).contiguous(), host


def uses_own_engine(shape, dtype=torch.float64):
    """True when this shape runs the hand-written FFT engine."""
    if isinstance(dtype, np.dtype) or dtype in (np.float64, np.float32):
        dtype = torch.float64 if np.dtype(dtype) == np.float64 else torch.float32
    return _plan(shape, dtype).own


def rfftn(x, s=None, axes=None, workers=None):
    """scipy.fft.rfftn over all axes (s must be None or x.shape)."""
    if not isinstance(x, torch.Tensor):
        x = np.asarray(x)
        if x.dtype not in (np.float32, np.float64):
            x = x.astype(np.float64)
    _check_axes(x, s, axes)
    if s is not None and tuple(s) != tuple(x.shape):
        raise ValueError("rfftn: zero-padding/cropping (s != x.shape) is not supported")
    t, host = _to_device(x, (torch.float64, torch.float32))
    shape = tuple(t.shape)
    p = _plan(shape, t.dtype)
    out = torch.empty(shape[:-1] + (shape[-1] // 2 + 1,), dtype=_CPLX[t.dtype], device=t.device)
    N.call("sfb_rfftn", p.handle, ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(out.data_ptr()), stream_ptr())
    return out.cpu().numpy() if host else out


def irfftn(x, s=None, axes=None, workers=None):
    """scipy.fft.irfftn over all axes; ``s`` is the real output shape (its
    last extent defaults to 2 (m - 1) like scipy)."""
    if not isinstance(x, torch.Tensor):
        x = np.asarray(x)
        if x.dtype not in (np.complex64, np.complex128):
            x = x.astype(np.complex128)
    _check_axes(x, s, axes)
    t, host = _to_device(x, (torch.complex128, torch.complex64))
    if s is None:
        s = tuple(t.shape[:-1]) + (2 * (t.shape[-1] - 1),)
    s = tuple(int(v) for v in s)
    if s[:-1] != tuple(t.shape[:-1]) or s[-1] // 2 + 1 != t.shape[-1]:
        raise ValueError("irfftn: zero-padding/cropping (s inconsistent with the input) is not supported")
    rdt = _REAL[t.dtype]
    p = _plan(s, rdt)
    out = torch.empty(s, dtype=rdt, device=t.device)
    N.call("sfb_irfftn", p.handle, ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(out.data_ptr()), stream_ptr())
    return out.cpu().numpy() if host else out
