"""dec3 cycle-counter probe (timing experiments only).  Needs the POLY_PROBE
library variant:
  POLY_VARIANT_FLAGS=-DPOLY_PROBE POLY_VARIANT_NAME=probe python paper_1805_01844_b200/_build.py
  POLY_LIB=paper_1805_01844_b200/libpolycomp_probe.so python profiles/probe_run.py --config 5
Prints the consumer / producer cycle split of the decompress pass-2 kernel."""
import argparse
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1805_01844_b200 import polycomp as pc  # noqa: E402
import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--reps", type=int, default=3)
args = ap.parse_args()
lib = pc.load_library()
c = workloads.config(args.config)
x = workloads.generate(args.config, seed=0, device="cuda")
out, nb = pc.poly_compress(x, c.block_len)
nbytes = int(nb.item())
dt = 16 if c.dtype == torch.uint16 else 32
pc.poly_decompress(out, nbytes, dt, c.n, c.block_len)
torch.cuda.synchronize()
assert lib.poly_probe_reset() == 0
for _ in range(args.reps):
    y, st = pc.poly_decompress(out, nbytes, dt, c.n, c.block_len)
torch.cuda.synchronize()
assert int(st.item()) == 0 and torch.equal(x, y)
buf = np.zeros(24, dtype=np.uint64)
assert lib.poly_probe_dump(buf.ctypes.data_as(ctypes.c_void_p)) == 0
b = buf.astype(np.float64)
names = {1: "full wait", 2: "decode (fast path)", 3: "copy out (fast path)"}
print("cfg%d consumers: total %.3g cycles; units %d" % (args.config, b[0], int(b[7])))
for i, nm in names.items():
    print("  %-22s %5.1f %%" % (nm, 100 * b[i] / b[0]))
print("  %-22s %5.1f %%" % ("other", 100 * (b[0] - b[1] - b[2] - b[3]) / b[0]))
print("producer: total %.3g cycles; waits (slot / ring) %.1f %%" % (b[4], 100 * b[5] / max(b[4], 1)))

# compress (poly_cmp3.cuh): counters 8..17
assert lib.poly_probe_reset() == 0
for _ in range(args.reps):
    out, nb = pc.poly_compress(x, c.block_len)
torch.cuda.synchronize()
assert lib.poly_probe_dump(buf.ctypes.data_as(ctypes.c_void_p)) == 0
b = buf.astype(np.float64)
if b[8] > 0:
    print("cfg%d compress consumers: total %.3g cycles; blocks %d" % (args.config, b[8], int(b[17])))
    for i, nm in {9: "fill wait", 10: "minmax + header", 11: "pack"}.items():
        print("  %-22s %5.1f %%" % (nm, 100 * b[i] / b[8]))
    print("  %-22s %5.1f %%" % ("other", 100 * (b[8] - b[9] - b[10] - b[11]) / b[8]))
    print("  writers: total %.3g; packed wait %.1f %%, prefix %.1f %%, copy+rest %.1f %%" % (
        b[12], 100 * b[13] / b[12], 100 * b[14] / b[12], 100 * (b[12] - b[13] - b[14]) / b[12]))
    print("  producer: total %.3g; empty wait %.1f %%" % (b[16], 100 * b[15] / max(b[16], 1)))
