"""Upper-bound experiment for binning map-0 blocks by base (timing only): the
same cfg2 blocks, once in generation order and once reordered so that blocks
of equal B (hence equal k, t and word count) are adjacent and a warp's 32 lanes
decode alike.  Prints compress / decompress GB/s for both orders.
usage: python profiles/sorted_blocks.py [--config 2] [--steps 20]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_01844_b200 import polycomp as pc  # noqa: E402
import workloads  # noqa: E402


def timed(x, L, steps):
    n = x.numel()
    dt = 16 if x.dtype == torch.uint16 else 32
    out, nb = pc.poly_compress(x, L)
    nbytes = int(nb.item())
    ws = pc.alloc_workspace(n, dt, L, x.device)
    y = torch.empty_like(x)
    st = torch.zeros(1, dtype=torch.int32, device=x.device)
    s = torch.cuda.current_stream()
    for _ in range(3):
        pc.poly_compress(x, L, out=out, compressed_bytes=nb, workspace=ws)
        pc.poly_decompress(out, nbytes, dt, n, L, out=y, status=st, workspace=ws)
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    for e in ev:
        e[0].record(s)
        pc.poly_compress(x, L, out=out, compressed_bytes=nb, workspace=ws)
        e[1].record(s)
        pc.poly_decompress(out, nbytes, dt, n, L, out=y, status=st, workspace=ws)
        e[2].record(s)
    torch.cuda.synchronize()
    assert int(st.item()) == 0 and torch.equal(x, y)
    c = sum(e[0].elapsed_time(e[1]) for e in ev) / steps
    d = sum(e[1].elapsed_time(e[2]) for e in ev) / steps
    b = n * x.element_size()
    return b / c / 1e6, b / d / 1e6, nbytes


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    pc.poly_init()
    c = workloads.config(args.config, 1.0)
    L = c.block_len
    x = workloads.generate(args.config, 1.0, 0, "cuda")
    nbk = x.numel() // L
    xi = x.view(torch.int16 if x.dtype == torch.uint16 else torch.int32)
    blk = xi[: nbk * L].view(nbk, L).to(torch.int32) & (0xffff if x.dtype == torch.uint16 else -1)
    B = blk.max(1).values - blk.min(1).values + 1
    # k = max{k : B^k <= 2^64} (approximate in fp64; the order is all that matters)
    k = torch.floor(64.0 / torch.log2(B.clamp(min=2).double()) + 1e-9).to(torch.int64)

    def reorder(key):
        order = torch.argsort(key, stable=True)
        xs = x.clone()
        xs.view(xi.dtype)[: nbk * L] = xi[: nbk * L].view(nbk, L)[order].reshape(-1)
        return xs

    for name, v in (("generation order", x), ("sorted by k", reorder(k)), ("sorted by B", reorder(B))):
        cg, dg, nbytes = timed(v, L, args.steps)
        print("%-18s compress %7.1f GB/s  decompress %7.1f GB/s  stream %d B" % (name, cg, dg, nbytes))


if __name__ == "__main__":
    main()
