"""Operator/plugin surface of the reference, on the device.

Mirror of ``batchbleu._backend`` (pkg/src/batchbleu/_backend.py:1-57).  The
reference dispatches to a Cython CPU kernel module or a numpy fallback; here
there is exactly one backend, ``cuda`` (``libtensorbleu_b200.so``), and no
CPU fallback — selecting the reference's CPU backends raises.

Every function accepts host arrays (numpy / CPU tensors; results come back
as numpy, like the reference) or CUDA tensors (results stay on the device).
These functions synchronise once to surface data-dependent errors with the
reference's exception types.
"""

from __future__ import annotations

import os

import numpy as np
import torch

from . import _native

NAME = "cuda"
_active = NAME


def available_backends() -> list[str]:
    """_backend.py:19-24.  Only the CUDA backend exists."""
    return [NAME]


def use_backend(name: str) -> None:
    """_backend.py:26-38: 'auto' and 'cuda' select the CUDA kernels; the
    reference's CPU backends do not exist here."""
    global _active
    if name in ("auto", NAME):
        _active = NAME
    elif name in ("python", "compiled"):
        raise RuntimeError(
            f"backend {name!r} is a CPU backend of the reference; this package only has 'cuda'")
    else:
        raise ValueError(f"unknown backend {name!r}")


def backend_name() -> str:
    return _active


def _device_for(*xs) -> tuple[bool, torch.device]:
    for x in xs:
        if isinstance(x, torch.Tensor) and x.is_cuda:
            return False, x.device
    return True, _native.require_cuda()


def _dev(x, dtype: torch.dtype, device: torch.device) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=dtype).contiguous()
    np_dt = {torch.int64: np.int64, torch.int32: np.int32}[dtype]
    return torch.from_numpy(np.ascontiguousarray(x, dtype=np_dt)).to(device)


def _flags(device: torch.device) -> torch.Tensor:
    return torch.zeros(1, dtype=torch.int32, device=device)


def unique_rows(rows):
    """Deduplicate the rows of a (T, n) int64 array (_backend.py:45-46,
    _kernels.pyx:36-81).

    Returns (unique (U, n), inverse (T,)), identical to the reference
    backends: unique rows in lexicographic order (signed int64), inverse the
    rank of each row's group (device: a hash dictionary, then an LSD radix
    sort of the unique rows, plugin.cu)."""
    lib = _native.load()
    host, device = _device_for(rows)
    if not isinstance(rows, torch.Tensor):
        rows = np.asarray(rows, dtype=np.int64)
    if rows.ndim != 2:
        raise ValueError(f"rows must be 2-D, got {rows.ndim} dimensions")
    t, n = int(rows.shape[0]), int(rows.shape[1])
    with torch.cuda.device(device):
        r = _dev(rows, torch.int64, device)
        uniq = torch.empty((t, n), dtype=torch.int64, device=device)
        inv = torch.empty(t, dtype=torch.int64, device=device)
        cnt = torch.zeros(1, dtype=torch.int64, device=device)
        wsb = lib.tb_unique_rows_workspace_bytes(t, n)
        ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=device)
        rc = lib.tb_unique_rows(r.data_ptr(), t, n, uniq.data_ptr(), inv.data_ptr(), cnt.data_ptr(),
                                ws.data_ptr(), ws.numel(), _native.stream_handle(device))
        _native.check(rc, "tb_unique_rows")
        u = int(cnt.item())
    uniq = uniq[:u]
    if host:
        return uniq.cpu().numpy(), inv.cpu().numpy()
    return uniq, inv


def _segment_call(fn_name, ids, seg_lengths, num_unique, ref_max=None):
    lib = _native.load()
    host, device = _device_for(ids, seg_lengths, ref_max)
    if not isinstance(seg_lengths, torch.Tensor):
        seg_lengths = np.asarray(seg_lengths, dtype=np.int64)
    if not isinstance(ids, torch.Tensor):
        ids = np.asarray(ids, dtype=np.int64).reshape(-1)
    b = int(seg_lengths.shape[0])
    u = int(num_unique)
    with torch.cuda.device(device):
        i = _dev(ids, torch.int64, device)
        s = _dev(seg_lengths, torch.int64, device)
        flags = _flags(device)
        wsb = lib.tb_segment_workspace_bytes(b, u)
        ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=device)
        if fn_name == "bincount":
            out = torch.empty((b, u), dtype=torch.int32, device=device)
            rc = lib.tb_segment_bincount(i.data_ptr(), i.numel(), s.data_ptr(), b, u, out.data_ptr(),
                                         flags.data_ptr(), ws.data_ptr(), ws.numel(),
                                         _native.stream_handle(device))
        else:
            rm = _dev(ref_max, torch.int32, device)
            if rm.dim() != 2 or rm.shape[0] != b:
                raise ValueError("ref_max row count does not match segment count")
            out = torch.empty(b, dtype=torch.int64, device=device)
            rc = lib.tb_clipped_numerators(i.data_ptr(), i.numel(), s.data_ptr(), b, rm.data_ptr(), u,
                                           out.data_ptr(), flags.data_ptr(), ws.data_ptr(), ws.numel(),
                                           _native.stream_handle(device))
        _native.check(rc, f"tb_{fn_name}")
        _native.raise_flags(int(flags.item()), f" [0, {u})")
    return out.cpu().numpy() if host else out


def segment_bincount(ids, seg_lengths, num_unique):
    """_backend.py:49-50 / _kernels.pyx:84-126: (B, U) int32 counts."""
    return _segment_call("bincount", ids, seg_lengths, num_unique)


def clipped_numerators(ids, seg_lengths, ref_max):
    """_backend.py:53-54 / _kernels.pyx:129-180: (B,) int64 clipped sums."""
    u = int(ref_max.shape[1]) if getattr(ref_max, "ndim", 0) == 2 else 0
    return _segment_call("clipped", ids, seg_lengths, u, ref_max=ref_max)


def count_binary(a, b, op: str):
    """Elementwise max ('max') / min ('min') of two int32 count matrices."""
    lib = _native.load()
    host, device = _device_for(a, b)
    with torch.cuda.device(device):
        x = _dev(a, torch.int32, device)
        y = _dev(b, torch.int32, device)
        out = torch.empty_like(x)
        rc = lib.tb_count_binary(x.data_ptr(), y.data_ptr(), out.data_ptr(), x.numel(),
                                 0 if op == "max" else 1, _native.stream_handle(device))
        _native.check(rc, "tb_count_binary")
    return out.cpu().numpy() if host else out


use_backend(os.environ.get("BATCHBLEU_BACKEND", "auto")
            if os.environ.get("BATCHBLEU_BACKEND", "auto") in ("auto", NAME) else "auto")
