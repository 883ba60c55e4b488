"""Padded batches of integer token IDs with explicit per-sequence lengths.

Mirror of ``batchbleu.batch.TokenBatch`` (pkg/src/batchbleu/batch.py:11-60):
same constructor, validation rules, error messages, ``from_lists`` and
``rows``.  In addition to numpy arrays / nested lists, ``ids`` may be a torch
tensor (int32 or int64).  CUDA tensors stay on the device (no copy) and are
validated by the ``tb_validate_batch`` kernel; host data is validated on the
host exactly like the reference.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import _native


def _is_torch(x) -> bool:
    return isinstance(x, torch.Tensor)


@dataclass(frozen=True)
class TokenBatch:
    """A (B, L) array of token IDs plus a (B,) array of valid lengths.

    Positions at or beyond ``lengths[i]`` in row ``i`` are padding and may
    hold any fill value; nothing downstream may depend on them
    (batch.py:13-17).
    """

    ids: object
    lengths: object

    def __post_init__(self):
        if _is_torch(self.ids) and self.ids.is_cuda:
            self._init_device()
            return
        if _is_torch(self.ids):
            self._init_host_torch()
            return
        # batch.py:22-37, verbatim semantics
        ids = np.ascontiguousarray(self.ids, dtype=np.int64)
        lengths = np.ascontiguousarray(
            self.lengths.cpu().numpy() if _is_torch(self.lengths) else self.lengths,
            dtype=np.int64)
        _validate_host(ids, lengths)
        object.__setattr__(self, "ids", ids)
        object.__setattr__(self, "lengths", lengths)

    # -- host torch tensors (e.g. pinned memory for the H2D path) -------------
    def _init_host_torch(self):
        ids = self.ids
        if ids.dtype not in (torch.int32, torch.int64):
            ids = ids.to(torch.int64)
        if ids.dim() != 2:
            raise ValueError(f"ids must be 2-D, got shape {tuple(ids.shape)}")
        if ids.stride(-1) != 1:
            ids = ids.contiguous()
        lengths = self.lengths
        lengths = (lengths.to(torch.int64) if _is_torch(lengths)
                   else torch.as_tensor(np.asarray(lengths, dtype=np.int64)))
        if lengths.is_cuda:
            lengths = lengths.cpu()
        _validate_host(ids.numpy(), lengths.numpy())
        object.__setattr__(self, "ids", ids)
        object.__setattr__(self, "lengths", lengths)

    # -- device tensors: validated on the GPU -----------------------------------
    def _init_device(self, validate: bool = True):
        ids = self.ids
        if ids.dtype not in (torch.int32, torch.int64):
            ids = ids.to(torch.int64)
        if ids.dim() != 2:
            raise ValueError(f"ids must be 2-D, got shape {tuple(ids.shape)}")
        if ids.stride(-1) != 1 or (ids.shape[0] > 1 and ids.stride(0) < ids.shape[1]):
            ids = ids.contiguous()
        lengths = self.lengths
        lengths = (lengths.to(device=ids.device, dtype=torch.int64) if _is_torch(lengths)
                   else torch.as_tensor(np.asarray(lengths, dtype=np.int64), device=ids.device))
        lengths = lengths.contiguous()
        if tuple(lengths.shape) != (ids.shape[0],):
            raise ValueError(
                f"lengths shape {tuple(lengths.shape)} does not match batch size {ids.shape[0]}")
        object.__setattr__(self, "ids", ids)
        object.__setattr__(self, "lengths", lengths)
        if validate and ids.shape[0] > 0:
            lib = _native.load()
            flag = torch.zeros(1, dtype=torch.int32, device=ids.device)
            with torch.cuda.device(ids.device):
                rc = lib.tb_validate_batch(
                    ids.element_size(), ids.data_ptr(), ids.stride(0) if ids.shape[0] > 1 else ids.shape[1],
                    ids.shape[1], lengths.data_ptr(), ids.shape[0], flag.data_ptr(),
                    _native.stream_handle(ids.device))
            _native.check(rc, "tb_validate_batch")
            _native.raise_flags(int(flag.item()))

    @classmethod
    def trusted(cls, ids: torch.Tensor, lengths: torch.Tensor) -> "TokenBatch":
        """Wrap device tensors WITHOUT the validation pass (no host sync).

        For training loops whose token IDs are known-good.  The kernels still
        clamp lengths and flag bad data, so nothing reads out of bounds."""
        obj = object.__new__(cls)
        object.__setattr__(obj, "ids", ids)
        object.__setattr__(obj, "lengths", lengths)
        if not (_is_torch(ids) and ids.is_cuda):
            raise ValueError("TokenBatch.trusted expects CUDA tensors")
        obj._init_device(validate=False)
        return obj

    def _row_view(self, want64: bool):
        """(ids pointer, ld, width, lengths pointer, token bytes) of this batch
        for the C ABI, plus the arrays that keep those pointers alive.  The view
        of the batch's own arrays is cached (they are read live on every call:
        in-place writes to a trusted buffer are seen).  When `want64` widens
        int32 IDs (batches of one call share a token width) the copy is made
        per call and never cached, so it cannot go stale."""
        ids, lengths = self.ids, self.lengths
        widen = want64 and (ids.dtype != np.int64 if isinstance(ids, np.ndarray) else ids.dtype != torch.int64)
        key = "_view"
        v = None if widen else self.__dict__.get(key)
        if v is not None:
            return v
        if isinstance(ids, np.ndarray):
            if want64 and ids.dtype != np.int64:
                ids = ids.astype(np.int64)
            ptr, isz, ld = ids.ctypes.data, ids.itemsize, ids.strides[0] // ids.itemsize
        else:
            if want64 and ids.dtype != torch.int64:
                ids = ids.to(torch.int64)
            ptr, isz, ld = ids.data_ptr(), ids.element_size(), ids.stride(0)
        if ids.shape[0] <= 1:
            ld = ids.shape[1]
        lptr = lengths.ctypes.data if isinstance(lengths, np.ndarray) else lengths.data_ptr()
        v = ((ptr, ld, int(ids.shape[1]), lptr, isz), (ids, lengths))
        if not widen:
            object.__setattr__(self, key, v)
        return v

    @property
    def batch_size(self) -> int:
        v = self.__dict__.get("_bs")  # cached: the batch is immutable (per-call overhead)
        if v is None:
            v = int(self.ids.shape[0])
            object.__setattr__(self, "_bs", v)
        return v

    @property
    def _tok32(self) -> bool:
        """Token IDs are int32 (numpy or torch), cached."""
        v = self.__dict__.get("_t32")
        if v is None:
            dt = self.ids.dtype
            v = (dt is torch.int32) if isinstance(dt, torch.dtype) else (dt == np.int32)
            object.__setattr__(self, "_t32", v)
        return v

    @property
    def max_len(self) -> int:
        return int(self.ids.shape[1])

    @property
    def is_device(self) -> bool:
        v = self.__dict__.get("_dev")
        if v is None:
            v = _is_torch(self.ids) and self.ids.is_cuda
            object.__setattr__(self, "_dev", v)
        return v

    @classmethod
    def from_lists(cls, sentences: Sequence[Sequence[int]], pad_value: int = 0,
                   min_width: int = 0) -> "TokenBatch":
        """Pack variable-length ID lists into a padded batch (batch.py:47-56)."""
        lengths = np.array([len(s) for s in sentences], dtype=np.int64)
        width = max(int(lengths.max(initial=0)), min_width)
        ids = np.full((len(sentences), width), pad_value, dtype=np.int64)
        for i, s in enumerate(sentences):
            ids[i, : len(s)] = s
        return cls(ids=ids, lengths=lengths)

    def rows(self) -> list[list[int]]:
        """Valid tokens per sentence, as plain lists (batch.py:58-60)."""
        ids = self.ids.cpu().numpy() if _is_torch(self.ids) else self.ids
        lengths = self.lengths.cpu().numpy() if _is_torch(self.lengths) else self.lengths
        return [ids[i, : lengths[i]].tolist() for i in range(self.batch_size)]


def _validate_host(ids: np.ndarray, lengths: np.ndarray) -> None:
    """batch.py:25-35: same checks, order and messages; the element checks run
    in the native library on its host threads (tb_validate_host)."""
    if ids.ndim != 2:
        raise ValueError(f"ids must be 2-D, got shape {ids.shape}")
    if lengths.shape != (ids.shape[0],):
        raise ValueError(
            f"lengths shape {lengths.shape} does not match batch size {ids.shape[0]}")
    if ids.shape[0] == 0:
        return
    if ids.dtype not in (np.int32, np.int64) or not ids.flags.c_contiguous and ids.strides[1] != ids.itemsize:
        ids = np.ascontiguousarray(ids, dtype=np.int64)
    lengths = np.ascontiguousarray(lengths, dtype=np.int64)
    ld = ids.strides[0] // ids.itemsize if ids.shape[0] > 1 else ids.shape[1]
    rc = _native.load().tb_validate_host(ids.itemsize, ids.ctypes.data, ld, ids.shape[1],
                                         lengths.ctypes.data, ids.shape[0])
    if rc < 0:
        _native.check(-rc, "tb_validate_host")
    if rc & _native.TB_FLAG_BAD_LENGTH:
        raise ValueError("lengths must lie in [0, max_len]")
    if rc & _native.TB_FLAG_NEGATIVE_ID:
        raise ValueError("token IDs within valid positions must be non-negative")
