"""Break down the host-side overhead of one small sentence_bleu call (GPU box)."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2510_05485_b200 as tb  # noqa: E402
from paper_2510_05485_b200 import _native, bleu  # noqa: E402


def t(fn, reps=200):
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return f"median {1e6 * np.median(ts):7.2f} us  min {1e6 * np.min(ts):7.2f} us"


def main():
    cid = torch.randint(0, 100, (1, 8)).pin_memory()
    cl = torch.tensor([8])
    cand = tb.TokenBatch(ids=cid, lengths=cl)
    refs = [tb.TokenBatch(ids=cid, lengths=cl)]
    cfg = tb.BleuConfig()
    lib = _native.load()
    dev = torch.device("cuda", 0)
    print("require_cuda          ", t(lambda: _native.require_cuda()))
    print("stream_handle         ", t(lambda: _native.stream_handle(dev)))
    print("row views x2 (cached) ", t(lambda: [b._row_view(True) for b in (cand, refs[0])]))
    print("sentence_bleu (tiny)  ", t(lambda: tb.sentence_bleu(cand, refs, cfg)))
    v = cand._row_view(True)[0]
    out = np.empty(1)
    flags = ctypes.c_int32(0)
    w = bleu._weights_arg(cfg)
    s = _native.stream_handle(dev)
    ra = (ctypes.c_void_p * 1)(v[0])
    rl = (ctypes.c_int64 * 1)(8)
    rw = (ctypes.c_int64 * 1)(8)
    rn = (ctypes.c_void_p * 1)(v[3])

    def raw():
        lib.tb_bleu_host(8, v[0], 8, 8, v[3], 1, ra, rl, rw, rn, 1, 4, 0, 0.1, 1.0, w,
                         None, None, None, None, out.ctypes.data, None, None, None, None,
                         ctypes.byref(flags), s)
    print("tb_bleu_host raw      ", t(raw))
    dc = torch.zeros(1, 8, dtype=torch.int64, device=dev)
    dl = torch.full((1,), 8, dtype=torch.int64, device=dev)
    dout = torch.empty(1, dtype=torch.float64, device=dev)
    dflag = torch.zeros(1, dtype=torch.int32, device=dev)
    ws = _native.workspace.get(dev, 1 << 16)
    da = (ctypes.c_void_p * 1)(dc.data_ptr())
    dn = (ctypes.c_void_p * 1)(dl.data_ptr())

    def raw_dev():
        lib.tb_bleu_stats(8, dc.data_ptr(), 8, 8, dl.data_ptr(), 1, da, rl, rw, dn, 1, 4, 0, 0.1, 1.0, w,
                          None, None, None, None, dout.data_ptr(), None, None, None, None,
                          dflag.data_ptr(), ws.data_ptr(), ws.numel(), s)

    print("tb_bleu_stats launch  ", t(raw_dev))
    print("tb_bleu_stats + sync  ", t(lambda: (raw_dev(), torch.cuda.synchronize())))
    print("empty sync            ", t(lambda: torch.cuda.synchronize()))
    x = torch.zeros(1, device=dev)
    print("tiny torch kernel+sync", t(lambda: (x.add_(1), torch.cuda.synchronize())))


if __name__ == "__main__":
    main()
