"""Per-phase timing of the fused kernel (debug build with -DTB_PHASES).

    python tools/phase_profile.py [--workload c2]

Loads libtensorbleu_b200_phases.so instead of the product library, runs the
workload, and prints for every phase mark the median / p90 time since the
CTA started, plus the spread of CTA start/finish times (ns, %globaltimer)."""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_05485_b200 import _native  # noqa: E402

_native.LIB_PATH = os.path.join(_native.PKG_DIR, "libtensorbleu_b200_phases.so")
import paper_2510_05485_b200 as tb  # noqa: E402
import bench  # noqa: E402

NAMES = {0: "start", 1: "lengths", 2: "staged", 28: "o1.claims", 29: "o1.verify", 3: "o1.inserted", 26: "o1.lookup", 4: "o1.live", 30: "epilogue", 31: "finish"}
for n in range(2, 7):
    for k, nm in enumerate(["P0clear", "P1cand", "P2ref", "P3live"]):
        NAMES.setdefault(3 + 4 * (n - 1) + k, f"o{n}.{nm}")
NAMES[24] = "orders>=2"
NAMES[1] = "epi.stores"
NAMES[23] = "epi.math"
NAMES.update({20: "f.bitmaps", 21: "f.filter", 22: "f.match"})


def build():
    import subprocess
    sys.path.insert(0, ROOT)
    import __graft_entry__ as g
    out = os.path.join(_native.PKG_DIR, "libtensorbleu_b200_phases.so")
    subprocess.check_call([g._nvcc(), *g.NVCC_FLAGS, "-DTB_PHASES", *g.SOURCES, "-o", out], cwd=g.CSRC)


def main():
    if "--build" in sys.argv:
        build()
        return
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="c2")
    ap.add_argument("--dtype", default="int32")
    ap.add_argument("--data", default="uniform")
    args = ap.parse_args()
    b, l, v, r, sm = bench.WORKLOADS[args.workload][:5]
    (cid, clen), refs = bench.generate_batch(b, l, v, r, data=args.data)
    dt = torch.int32 if args.dtype == "int32" else torch.int64
    cand = tb.TokenBatch(ids=torch.as_tensor(cid).cuda().to(dt), lengths=torch.as_tensor(clen).cuda())
    rb = [tb.TokenBatch(ids=torch.as_tensor(i).cuda().to(dt), lengths=torch.as_tensor(ln).cuda()) for i, ln in refs]
    lib = _native.load()
    lib.tb_debug_phase_buffer.argtypes = [ctypes.c_void_p]
    buf = torch.zeros(b * 32, dtype=torch.int64, device="cuda")
    lib.tb_debug_phase_buffer(buf.data_ptr())
    plan = tb.SentenceBleuPlan(cand, rb, tb.BleuConfig(smoothing=sm))
    # launch through the instrumented library (the plan's own launches go
    # through _hostpath, which is linked against the product library)
    views, B, N, smc, eps, k, waddr, outs, err, ws, wsb = plan._launch_args
    P = ctypes.c_void_p
    R = len(views) - 1
    args = (views[0][4], views[0][0], views[0][1], views[0][2], views[0][3], R,
            (P * R)(*[v[0] for v in views[1:]]), (ctypes.c_int64 * R)(*[v[1] for v in views[1:]]),
            (ctypes.c_int64 * R)(*[v[2] for v in views[1:]]), (P * R)(*[v[3] for v in views[1:]]),
            B, N, smc, eps, k, waddr, *outs, err, ws, wsb)

    def run():
        rc = lib.tb_bleu_stats(*args, torch.cuda.current_stream().cuda_stream)
        assert rc == 0, rc

    for _ in range(5):
        run()
    buf.zero_()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    flush.zero_()
    run()
    torch.cuda.synchronize()
    t = buf.cpu().numpy().reshape(b, 32).astype(np.int64)
    grid = int((t[:, 0] > 0).sum())
    t = t[:grid]
    t0 = t[:, 0].min()
    print(f"CTAs {grid}; CTA start spread {np.ptp(t[:, 0])} ns; first start -> last finish "
          f"{t[:, 31].max() - t0} ns")
    print(f"order-1 deferred inserts per CTA: mean {t[:, 27].mean():.1f} max {t[:, 27].max()}")
    print(f"filter passes per CTA: mean {t[:, 25].mean():.1f} max {t[:, 25].max()}")
    t[:, 27] = 0
    t[:, 25] = 0
    for k in [0, 1, 2, 20, 21, 22, 28, 29, 3, 26, 4] + list(range(5, 20)) + [23, 24, 30, 31]:
        col = t[:, k]
        ok = col > 0
        if not ok.any():
            continue
        rel = col[ok] - t[ok, 0]
        print(f"{NAMES.get(k, k):>12}: n={ok.sum():4d} since CTA start median {np.median(rel):8.0f} "
              f"p90 {np.percentile(rel, 90):8.0f} max {rel.max():8.0f} ns")


if __name__ == "__main__":
    main()
