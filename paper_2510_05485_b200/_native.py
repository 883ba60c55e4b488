"""ctypes binding of the C ABI in include/tensorbleu.h.

The shared library ``libtensorbleu_b200.so`` is built in-tree by
``__graft_entry__.build()`` (nvcc, sm_100a).  There is no CPU fallback: if
the library or a CUDA device is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading
from typing import Optional

import torch

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_NAME = "libtensorbleu_b200.so"
LIB_PATH = os.path.join(PKG_DIR, LIB_NAME)
HEADER_PATH = os.path.join(os.path.dirname(PKG_DIR), "include", "tensorbleu.h")

TB_OK = 0
TB_ERR_INVALID_ARG = 1
TB_ERR_CAPACITY = 2
TB_ERR_CUDA = 3
TB_ERR_UNSUPPORTED = 4
TB_ERR_WORKSPACE = 5

TB_FLAG_BAD_LENGTH = 1
TB_FLAG_NEGATIVE_ID = 2
TB_FLAG_ID_RANGE = 4
TB_FLAG_SEGMENTS = 8

TB_MAX_ORDER = 32
TB_MAX_REFS = 32

SMOOTHING_CODES = {"none": 0, "floor": 1, "add-k": 2, "exp": 3}

_P = ctypes.c_void_p
_I32 = ctypes.c_int32
_I64 = ctypes.c_int64
_F64 = ctypes.c_double
_SZ = ctypes.c_size_t

# name -> (restype, argtypes)
SIGNATURES = {
    "tb_version": (ctypes.c_char_p, []),
    "tb_strerror": (ctypes.c_char_p, [ctypes.c_int]),
    "tb_last_cuda_error": (ctypes.c_char_p, []),
    "tb_bleu_workspace_bytes": (_SZ, [_I64, _I32, _I64, _P, _I32, _I32]),
    "tb_bleu_stats": (ctypes.c_int, [
        _I32,                      # token_bytes
        _P, _I64, _I64, _P,        # cand ids, ld, width, len
        _I32, _P, _P, _P, _P,      # R, ref ids[], ref ld[], ref width[], ref len[]
        _I64, _I32,                # batch, max_order
        _I32, _F64, _F64, _P,      # smoothing, eps, k, weights
        _P, _P, _P, _P,            # num, den, cand_len_out, eff_ref_out
        _P, _P, _P,                # scores, precisions, bp
        _P, _P,                    # totals, corpus
        _P,                        # err flag
        _P, _SZ, _P,               # workspace, bytes, stream
    ]),
    "tb_bleu_host": (ctypes.c_int, [
        _I32,                      # token_bytes
        _P, _I64, _I64, _P,        # cand ids, ld, width, len  (host or device)
        _I32, _P, _P, _P, _P,      # R, ref ids[], ref ld[], ref width[], ref len[]
        _I64, _I32,                # batch, max_order
        _I32, _F64, _F64, _P,      # smoothing, eps, k, weights
        _P, _P, _P, _P,            # num, den, cand_len_out, eff_ref_out   (host)
        _P, _P, _P,                # scores, precisions, bp                 (host)
        _P, _P,                    # totals, corpus                         (host)
        _P, _P,                    # flags_out (host int32), stream
    ]),
    "tb_bleu_scores": (ctypes.c_int, [_P, _P, _P, _P, _I64, _I32, _I32, _F64, _F64, _P,
                                      _P, _P, _P, _P]),
    "tb_bleu_totals": (ctypes.c_int, [_P, _P, _P, _P, _I64, _I32, _P, _P]),
    "tb_bleu_scores_any": (ctypes.c_int, [_P, _P, _P, _P, _I64, _I32, _I32, _F64, _F64, _P, _I32,
                                          _P, _P, _P, _P]),
    "tb_validate_batch": (ctypes.c_int, [_I32, _P, _I64, _I64, _P, _I64, _P, _P]),
    "tb_validate_host": (ctypes.c_int, [_I32, _P, _I64, _I64, _P, _I64]),
    "tb_windows_workspace_bytes": (_SZ, [_I64]),
    "tb_flatten_windows": (ctypes.c_int, [_I32, _P, _I64, _I64, _P, _I64, _I32, _P, _P, _P, _SZ, _P]),
    "tb_unique_rows_workspace_bytes": (_SZ, [_I64, _I32]),
    "tb_unique_rows": (ctypes.c_int, [_P, _I64, _I32, _P, _P, _P, _P, _SZ, _P]),
    "tb_segment_workspace_bytes": (_SZ, [_I64, _I64]),
    "tb_segment_bincount": (ctypes.c_int, [_P, _I64, _P, _I64, _I64, _P, _P, _P, _SZ, _P]),
    "tb_clipped_numerators": (ctypes.c_int, [_P, _I64, _P, _I64, _P, _I64, _P, _P, _P, _SZ, _P]),
    "tb_count_binary": (ctypes.c_int, [_P, _P, _P, _I64, _I32, _P]),
}

_lib = None
_lock = threading.Lock()


class NativeLibraryError(RuntimeError):
    """The CUDA library is not built or cannot be loaded."""


def load():
    """Load (once) and return the ctypes handle of the CUDA library."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryError(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


_hp = None


def hostpath():
    """The CPython binding of tb_bleu_host (built in-tree next to the library)."""
    global _hp
    if _hp is None:
        load()
        try:
            from . import _hostpath
        except ImportError as e:
            raise NativeLibraryError(f"the _hostpath extension is not built ({e}); run "
                                     "`python -c 'import __graft_entry__ as g; g.build()'`") from e
        _hp = _hostpath
    return _hp


_cuda_ok: Optional[bool] = None


def require_cuda_available() -> None:
    global _cuda_ok
    if _cuda_ok is None:
        _cuda_ok = torch.cuda.is_available()
    if not _cuda_ok:
        raise RuntimeError("paper_2510_05485_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")


def require_cuda(device: Optional[torch.device] = None) -> torch.device:
    global _cuda_ok
    if _cuda_ok is None:
        _cuda_ok = torch.cuda.is_available()
    if not _cuda_ok:
        raise RuntimeError("paper_2510_05485_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    device = torch.device(device)
    if device.type != "cuda":
        raise RuntimeError(f"expected a CUDA device, got {device}")
    if device.index is None:
        device = torch.device("cuda", torch.cuda.current_device())
    return device


def check(rc: int, what: str) -> None:
    """Map a TB_ERR_* code to the reference's exception types."""
    if rc == TB_OK:
        return
    lib = load()
    msg = f"{what}: {lib.tb_strerror(rc).decode()}"
    if rc == TB_ERR_CUDA:
        msg += f" ({lib.tb_last_cuda_error().decode()})"
    if rc in (TB_ERR_INVALID_ARG, TB_ERR_UNSUPPORTED):
        raise ValueError(msg)
    if rc == TB_ERR_CAPACITY:
        from .ngrams import CapacityError
        raise CapacityError(msg)
    raise RuntimeError(msg)


def raise_flags(flags: int, what: str = "") -> None:
    """Raise the reference's error for device-detected data errors."""
    if flags & TB_FLAG_BAD_LENGTH:
        raise ValueError("lengths must lie in [0, max_len]")               # batch.py:30-31
    if flags & TB_FLAG_NEGATIVE_ID:
        raise ValueError("token IDs within valid positions must be non-negative")  # batch.py:33-34
    if flags & TB_FLAG_SEGMENTS:
        raise ValueError("segment lengths do not sum to the number of IDs")  # _kernels.pyx:96-97
    if flags & TB_FLAG_ID_RANGE:
        raise ValueError(f"compact ID out of range{what}")                  # _kernels.pyx:124-125


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def current_device_index() -> int:
    """Index of torch's current CUDA device; raises without a GPU (no CPU fallback)."""
    require_cuda_available()
    return torch.cuda.current_device()


def raw_stream(index: int) -> int:
    """cudaStream_t of torch's current stream on device `index`."""
    if _raw_stream is not None:
        return _raw_stream(index)
    return torch.cuda.current_stream(index).cuda_stream


def stream_handle(device: torch.device) -> int:
    """cudaStream_t of torch's current stream on `device` (the cheap internal
    accessor when this torch build has it)."""
    if _raw_stream is not None:
        return _raw_stream(device.index if device.index is not None else torch.cuda.current_device())
    return torch.cuda.current_stream(device).cuda_stream


class _Workspace:
    """Per (device, stream) zero-initialised scratch owned by torch's allocator.

    The fused kernel leaves its corpus accumulators zeroed, so one
    torch.zeros at growth time is the only initialisation ever needed."""

    def __init__(self):
        self._bufs = {}
        self._lock = threading.Lock()

    def get(self, device: torch.device, nbytes: int) -> torch.Tensor:
        key = (device.index, stream_handle(device))
        with self._lock:
            buf = self._bufs.get(key)
            if buf is None or buf.numel() < nbytes:
                size = max(int(nbytes), 1 << 16)
                if buf is not None:
                    size = max(size, 2 * buf.numel())
                buf = torch.zeros(size, dtype=torch.uint8, device=device)
                self._bufs[key] = buf
            return buf


workspace = _Workspace()


def version() -> str:
    return load().tb_version().decode()
