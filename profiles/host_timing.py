"""Time poly_compress_host / poly_decompress_host (pinned buffers) on cfg2,
chunked (default) and serial (POLY_HOST_SERIAL=1), each call alone."""
import os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_01844_b200 import polycomp as pc  # noqa: E402
import workloads  # noqa: E402

x = workloads.generate(2, 1.0, 0, "cuda")
n, L, dt = x.numel(), 30, 16
h_in = torch.empty(n, dtype=x.dtype, pin_memory=True)
h_in.copy_(x.cpu())
cap = pc.poly_max_compressed_bytes(n, dt, L)
d_in = torch.empty(max(cap, 2 * n), dtype=torch.uint8, device="cuda")
d_out = torch.empty(max(cap, 2 * n), dtype=torch.uint8, device="cuda")
ws = pc.alloc_workspace(n, dt, L, d_in.device)
h_s = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=x.dtype, pin_memory=True)
for mode in ("chunked", "serial", "chunked"):
    if mode == "serial":
        os.environ["POLY_HOST_SERIAL"] = "1"
    else:
        os.environ.pop("POLY_HOST_SERIAL", None)
    nb = pc.poly_compress_host(h_in, L, d_in, d_out, ws, h_s)
    pc.poly_decompress_host(h_s, nb, dt, n, L, d_in, d_out, ws, h_out)
    tc = td = 0.0
    for _ in range(3):
        t0 = time.perf_counter(); nb = pc.poly_compress_host(h_in, L, d_in, d_out, ws, h_s); t1 = time.perf_counter()
        st = pc.poly_decompress_host(h_s, nb, dt, n, L, d_in, d_out, ws, h_out); t2 = time.perf_counter()
        tc += t1 - t0; td += t2 - t1
    print("%-8s compress_host %.2f ms  decompress_host %.2f ms  ok=%s" % (mode, tc / 3 * 1e3, td / 3 * 1e3,
          st == 0 and torch.equal(h_out, h_in)))
