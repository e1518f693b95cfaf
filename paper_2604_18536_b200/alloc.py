"""Allocation funnel with a counter (mirror of alloc.py:1-23).

Every field-sized device buffer the package creates goes through
:func:`zeros`, so tests can assert that the stepping loop allocates nothing
per step once its workspace exists.
"""

import numpy as np
import torch

_count = 0

_TORCH = {np.dtype(np.float64): torch.float64, np.dtype(np.float32): torch.float32}


def torch_dtype(dtype):
    return _TORCH[np.dtype(dtype)]


def zeros(shape, dtype, device=None):
    global _count
    _count += 1
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    return torch.zeros(tuple(shape), dtype=torch_dtype(dtype), device=device)


def empty(shape, dtype, device=None):
    """Uninitialised buffer for outputs a kernel writes completely."""
    global _count
    _count += 1
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    return torch.empty(tuple(shape), dtype=torch_dtype(dtype), device=device)


def allocation_count():
    return _count
