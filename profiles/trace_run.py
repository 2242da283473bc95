"""Pipeline event trace of one compress and one decompress call (timing
experiments only).  Needs the POLY_TRACE library variant:
  POLY_VARIANT_FLAGS=-DPOLY_TRACE POLY_VARIANT_NAME=trace python -c "from paper_1805_01844_b200 import _build; _build.build(force=True)"
  POLY_LIB=paper_1805_01844_b200/libpolycomp_trace.so python profiles/trace_run.py --config 2 --out gpurun_out/trace_cfg2
Writes <out>_c.npy / <out>_d.npy (CTA x tile x event globaltimer stamps, event
10 = tile id) and prints per-stage latency medians."""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_01844_b200 import polycomp as pc  # noqa: E402
import workloads  # noqa: E402

TILES, EV = 1024, 16
NAMES_C = {0: "ticket", 1: "in landed(w0)", 9: "minmax done(w0)", 11: "barrier 1 passed", 2: "AGG published",
           3: "ring alloc", 4: "pack done(w0)",
           8: "pack done(w15)", 5: "writer got rec", 6: "lookback done", 7: "copy done"}
NAMES_D = {0: "ticket", 1: "hdr landed", 2: "AGG published", 3: "LB start", 4: "lookback done", 5: "ring alloc",
           6: "payload landed(w0)", 9: "payload landed(w15)", 7: "w0 done", 8: "last warp done"}


def grab(lib):
    nb = lib.poly_trace_bytes()
    buf = np.empty(nb // 8, dtype=np.uint64)
    assert lib.poly_trace_dump(buf.ctypes.data_as(ctypes.c_void_p), ctypes.c_uint64(nb)) == 0
    return buf.reshape(-1, TILES, EV)


def report(tr, names, label, pairs):
    ok = tr[:, :, 0] != np.uint64(0xffffffffffffffff)
    t0 = tr[:, :, 0][ok].min()
    print("== %s: %d CTAs with tiles, %d tiles" % (label, int(ok.any(1).sum()), int(ok.sum())))
    valid = (tr != np.uint64(0xffffffffffffffff))
    for a, b in pairs:
        m = valid[:, :, a] & valid[:, :, b] & ok
        d = (tr[:, :, b][m].astype(np.int64) - tr[:, :, a][m].astype(np.int64)) / 1000.0
        if d.size:
            print("  %-22s -> %-22s  med %7.2f us  p10 %7.2f  p90 %7.2f" % (names[a], names[b], np.median(d),
                                                                           np.percentile(d, 10), np.percentile(d, 90)))
    # per-CTA tile period (steady state: middle half of each CTA's tiles)
    per = []
    for c in range(tr.shape[0]):
        n = int(ok[c].sum())
        if n > 8:
            ts = tr[c, :n, 0].astype(np.int64)
            per.append(np.median(np.diff(ts[n // 4: 3 * n // 4])) / 1000.0)
    if per:
        print("  tile period per CTA (ticket to ticket): med %.2f us" % np.median(per))
    # warp 0: from its pack end to the next tile's stage landing (input wait)
    if valid[:, :, 4].any() and valid[:, :, 1].any():
        g = []
        for c in range(tr.shape[0]):
            n = int(ok[c].sum())
            if n > 8:
                a4 = tr[c, n // 4: 3 * n // 4, 4].astype(np.int64)
                b1 = tr[c, n // 4 + 1: 3 * n // 4 + 1, 1].astype(np.int64)
                g.append(np.median(b1 - a4) / 1000.0)
        if g:
            print("  pack done(w0) -> next in landed(w0): med %.2f us" % np.median(g))
    end = max(int(tr[:, :, e][valid[:, :, e]].max()) for e in names if valid[:, :, e].any())
    print("  span first ticket -> last event: %.1f us" % ((end - int(t0)) / 1000.0))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--out", default="gpurun_out/trace")
    args = ap.parse_args()
    lib = pc.load_library()
    lib.poly_trace_bytes.restype = ctypes.c_uint64
    lib.poly_trace_dump.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
    cfg = workloads.config(args.config, args.scale)
    x = workloads.generate(args.config, args.scale, 0, "cuda")
    L = cfg.block_len or x.numel()
    out, nb = pc.poly_compress(x, L)
    torch.cuda.synchronize()
    dt = pc.POLY_U16 if x.dtype == torch.uint16 else pc.POLY_U32
    for _ in range(3):  # warm-up
        pc.poly_compress(x, L, out=out)
        pc.poly_decompress(out, int(nb.item()), dt, x.numel(), L)
    torch.cuda.synchronize()
    lib.poly_trace_reset()
    pc.poly_compress(x, L, out=out)
    torch.cuda.synchronize()
    tc = grab(lib)
    lib.poly_trace_reset()
    y, st = pc.poly_decompress(out, int(nb.item()), dt, x.numel(), L)
    torch.cuda.synchronize()
    td = grab(lib)
    for tag, tr in (("c", tc), ("d", td)):
        ok = tr[:, :, 0] != np.uint64(0xffffffffffffffff)
        nc, nt = int(ok.any(1).sum()), int(ok.sum(1).max())
        np.savez_compressed(args.out + "_%s.npz" % tag, tr=tr[:max(nc, 1), :max(nt, 1)])
    report(tc, NAMES_C, "compress", [(0, 1), (1, 9), (9, 11), (11, 2), (2, 3), (3, 4), (4, 8), (4, 5), (5, 6), (6, 7),
                                     (0, 7)])
    if (td[:, :, 0] != np.uint64(0xffffffffffffffff)).any():  # pipeline decompress (map 0) only
        report(td, NAMES_D, "decompress", [(0, 1), (1, 2), (2, 3), (3, 4), (4, 5), (5, 6), (6, 9), (6, 7), (7, 8), (0, 8)])


if __name__ == "__main__":
    main()
