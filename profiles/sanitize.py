"""Small round trips for compute-sanitizer (memcheck / racecheck / synccheck):
every regime and map once, bit-exact check against the oracle.
usage: compute-sanitizer --tool memcheck python profiles/sanitize.py"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_01844_b200 import polycomp as pc  # noqa: E402
from oracle import coracle  # noqa: E402

rng = np.random.default_rng(7)
cases = [
    (rng.integers(240, 270, 30 * 5000).astype(np.uint16), 30),      # map 0, several tiles
    (rng.integers(0, 4096, 1024 * 40).astype(np.uint16), 1024),     # map 1, G = 1
    (rng.integers(900, 1100, 4096 * 30).astype(np.uint16), 4096),   # map 1, G > 1
    (rng.integers(0, 1 << 20, 65536 * 300).astype(np.uint32), 65536),  # LARGE2
    (rng.integers(0, 300, 1 << 18).astype(np.uint16), 0),           # one block (LARGE)
    (rng.integers(0, 7, 31).astype(np.uint16), 3),                  # tiny, ragged
]
for x, L in cases:
    t = torch.from_numpy(x.view(np.int16 if x.dtype == np.uint16 else np.int32).copy())
    xd = t.view(torch.uint16 if x.dtype == np.uint16 else torch.uint32).cuda()
    Lb = L or x.size
    out, nb = pc.poly_compress(xd, Lb)
    nbytes = int(nb.item())
    ref = coracle.compress(x, Lb)
    assert out[:nbytes].cpu().numpy().tobytes() == ref, ("stream", x.dtype, x.size, L)
    dt = 16 if x.dtype == np.uint16 else 32
    y, st = pc.poly_decompress(out, nbytes, dt, x.size, Lb)
    torch.cuda.synchronize()
    yv = y.cpu().view(torch.int16 if dt == 16 else torch.int32).numpy().view(x.dtype)
    assert int(st.item()) == 0 and np.array_equal(yv, x), ("values", x.dtype, x.size, L)
    print("ok", x.dtype, x.size, L, flush=True)
print("all ok")
