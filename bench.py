#!/usr/bin/env python
"""Benchmark of the B200 polynomial-codec hot path (one JSON line on rank 0).

A step = one pass of the whole hot path over one batch: poly_compress then
poly_decompress of the BASELINE workload, inputs resident in HBM.  The
headline workload is cfg5 (BASELINE.json configs[4]: 4 GiB of u16, the full
compress + decompress round trip, the largest single-GPU configuration); the
line also carries every other config measured the same way ("configs").

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

Correctness gate (never report timings for incorrect output):
before any timing the GPU stream is compared byte for byte with the C
oracle's stream of the same input, and the round trip with the input; after
the timed steps the last step's stream, values and status are checked again.
value     = uncompressed bytes of all ranks x K / max-over-ranks device time of
            the K steps (GB/s, compress + decompress in series).
e2e       = the same metric through poly_compress_host / poly_decompress_host
            (pinned host buffers, H2D + D2H inside the timed region).
roofline  = the dominant kernel's algorithmic bytes (I + C, read + written)
            per launch / its CUDA-event duration, against MEASURED_PEAKS.json.
cpu_baseline = the C oracle (oracle/oracle.c, all host cores) on the FULL
            input of the same workload (rank 0, N = 1 only).
lzma      = PAPER.md Tables 1-2 "Poly + LZMA" pairing, reported only: Python
            lzma preset 1 over the first 64 MiB of the input, raw and after
            the GPU codec.
--impl reference times that oracle as the reference arm (full input).
Multi-GPU (torchrun): every rank compresses its own batch (seed = rank), no
data-path collective ("scaling": "weak"); only the timing max is reduced.
"""
from __future__ import annotations

import argparse
import json
import statistics
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "compress & decompress GB/s (uncompressed input) on 1 B200; % HBM roofline; ratio"
FALLBACK_HBM_GBS = 6650.0


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=100)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--config", type=int, default=5, choices=[1, 2, 3, 4, 5, 6])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--ref-seconds", type=float, default=60.0,
                   help="reference arm: stop repeating full-input oracle steps after this much CPU time")
    p.add_argument("--scale", type=float, default=1.0, help=argparse.SUPPRESS)
    p.add_argument("--only", action="store_true", help="the headline config only (no other configs, no lzma)")
    p.add_argument("--no-roundtrip-check", action="store_true",
                   help="POLY_TIMING variant libraries only (outputs wrong by design): skip the checks")
    return p.parse_args()


def dist_init(args):
    import torch
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    elif torch.cuda.is_available():
        torch.cuda.set_device(local)
    return rank, world, local


def reduce_max(vals, world, dev="cpu"):
    """Max over ranks of each timing (the job's time is its slowest rank's)."""
    import torch
    t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=dev)
    if world > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t.tolist()]


def job_gbs(world, in_bytes, steps, total_ms):
    """Whole-job throughput: every rank processed `in_bytes` per step (weak
    scaling, no data-path collective), timed by the slowest rank."""
    return world * in_bytes * steps / (total_ms * 1e-3) / 1e9


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)", d
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)", {}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._th = None

    def _sample(self):
        try:
            r = subprocess.run(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
            if r.returncode == 0 and r.stdout.strip():
                self.rows.append([c.strip() for c in r.stdout.strip().split(",")])
        except Exception:
            pass

    def _run(self):
        while not self._stop.is_set():
            self._sample()
            self._stop.wait(0.05)

    def __enter__(self):
        self._th = threading.Thread(target=self._run, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._th:
            self._th.join(timeout=10)
        self._sample()  # one more at the end of the timed region (short regions get >= 2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = sorted(float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit())
        mx = max((float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()), default=None)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            for nm, v in zip(names, r[4:8]):
                if v.strip().lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(self.rows)}


def oracle_full(x_np, L, threads):
    """The C oracle on the whole input: compress then decompress (timed), the
    round trip checked.  Returns (stream bytes, compress s, decompress s)."""
    import numpy as np
    from oracle import coracle
    t0 = time.perf_counter()
    ref = coracle.compress(x_np, L, threads=threads)
    t1 = time.perf_counter()
    y, st = coracle.decompress(ref, threads=threads)
    t2 = time.perf_counter()
    if st != 0 or not np.array_equal(y, x_np):
        raise SystemExit("oracle round trip failed")
    return ref, t1 - t0, t2 - t1


def single_thread_oracle(x_np, L, threads):
    """One thread on the first 1/threads of the blocks (the same per-thread
    work as the all-core figure)."""
    import numpy as np
    from oracle import coracle
    Lb = L or x_np.size
    n1 = max(Lb, (x_np.size // max(1, threads)) // Lb * Lb) if L else x_np.size
    x1 = x_np[:n1]
    t0 = time.perf_counter()
    s1 = coracle.compress(x1, L, threads=1)
    y1, st1 = coracle.decompress(s1, threads=1)
    t1 = time.perf_counter() - t0
    assert st1 == 0 and np.array_equal(y1, x1)
    return round(x1.nbytes / t1 / 1e9, 4), "first %d values, 1 thread" % n1


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args, rank, world):
    """Reference arm: the oracle (plain C, all host cores) on the FULL input of
    the workload, compress + decompress per step, as many steps as fit in
    --ref-seconds (at least one).  Rank 0 only."""
    if rank != 0:
        return
    import workloads
    from oracle import coracle
    scale = getattr(args, "scale", 1.0)  # < 1 only in the CPU tests of this path
    c = workloads.config(args.config, scale)
    import torch
    # the seeded generator runs on the GPU when there is one (same bytes as the
    # GPU arm's input; it holds none of the codec's arithmetic), else on the CPU
    gdev = "cuda" if torch.cuda.is_available() else "cpu"
    x = workloads.generate(args.config, scale=scale, seed=0, device=gdev).cpu().numpy()
    threads = coracle.default_threads()
    times = []
    t_begin = time.perf_counter()
    for i in range(max(1, args.steps)):
        _, tc, td = oracle_full(x, c.block_len, threads)
        times.append(tc + td)
        if time.perf_counter() - t_begin > args.ref_seconds:
            break
    per = sum(times) / len(times)
    gbs = x.nbytes / per / 1e9
    cb = {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": "oracle",
          "sample": "full input (%s, seed 0), compress+decompress, %d step(s), all host cores" % (c.description, len(times)),
          "cpu_model": cpu_model()}
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "GB/s", "n_gpus": args.gpus,
        "steps": len(times), "steps_requested": args.steps, "warmup": 0, "ms_per_step": round(1e3 * per, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "u16" if c.dtype == torch.uint16 else "u32",
        "data": "synthetic", "config": {"workload": c.name, "n": c.n, "block_len": c.block_len},
        "cpu_baseline": cb, "e2e": {"value": cb["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                                    "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def traffic_from_profiles(kernel_key: str):
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f).get(kernel_key)
    except Exception:
        return None


def measure(args, cfg, steps, rank, world, local, clocks=True, keep_input=False):
    """Generate config `cfg` on the GPU, gate it against the oracle, time
    `steps` compress + decompress steps.  Returns (record, extras)."""
    import numpy as np
    import torch
    import workloads
    from oracle import coracle
    from paper_1805_01844_b200 import polycomp as pc

    dev = torch.device("cuda", local)
    c = workloads.config(cfg, 1.0)
    dt = 16 if c.dtype == torch.uint16 else 32
    x = workloads.generate(cfg, scale=1.0, seed=rank, device=dev)
    n, L = c.n, c.block_len
    in_bytes = n * (dt // 8)
    cap = pc.poly_max_compressed_bytes(n, dt, L)
    out = torch.empty(cap, dtype=torch.uint8, device=dev)
    nb = torch.zeros(1, dtype=torch.int64, device=dev)
    ws = pc.alloc_workspace(n, dt, L, dev)
    y = torch.empty_like(x)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev) if in_bytes < 256 << 20 else None

    # ---- correctness gate: the stream equals the oracle's, the round trip the input
    pc.poly_compress(x, L, out=out, compressed_bytes=nb, workspace=ws)
    int_nbytes = int(nb.item())
    pc.poly_decompress(out, int_nbytes, dt, n, L, out=y, status=st, workspace=ws)
    torch.cuda.synchronize()
    threads = max(1, coracle.default_threads() // max(1, world))
    x_np = x.cpu().numpy()
    ref, t_oc, t_od = oracle_full(x_np, L, threads)
    check = not args.no_roundtrip_check
    ref_dev = torch.from_numpy(np.frombuffer(ref, dtype=np.uint8).copy()).to(dev)
    exact = len(ref) == int_nbytes and torch.equal(out[:int_nbytes], ref_dev)
    rt_ok = int(st.item()) == 0 and torch.equal(x, y)
    if check and not (exact and rt_ok):
        raise SystemExit("cfg%d: GPU output differs from the oracle (stream %s, round trip %s) on rank %d: "
                         "no timing reported" % (cfg, exact, rt_ok, rank))

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        pc.poly_compress(x, L, out=out, compressed_bytes=nb, workspace=ws)
        if ev is not None:
            ev[1].record(stream)
        pc.poly_decompress(out, int_nbytes, dt, n, L, out=y, status=st, workspace=ws)
        if ev is not None:
            ev[2].record(stream)

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    y.zero_()
    st.fill_(-1)
    clk = ClockSampler(local) if clocks else None
    if clk:
        clk.__enter__()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    if flush is None:
        t_start.record(stream)
        for i in range(steps):
            step(evs[i])
        t_end.record(stream)
        torch.cuda.synchronize()
        total_ms = t_start.elapsed_time(t_end)
    else:  # small input (cfg1): flush L2 between steps, time the steps only
        for i in range(steps):
            flush.fill_(i & 0xff)
            step(evs[i])
        torch.cuda.synchronize()
        total_ms = sum(e[0].elapsed_time(e[2]) for e in evs)
    if clk:
        clk.__exit__()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    # ---- the timed steps' output is checked again (the kernels race by design)
    post_ok = (int(nb.item()) == int_nbytes and torch.equal(out[:int_nbytes], ref_dev) and int(st.item()) == 0
               and torch.equal(x, y))
    if check and not post_ok:
        raise SystemExit("cfg%d: output of the timed steps differs from the oracle on rank %d" % (cfg, rank))
    del ref_dev
    comp_ms = [e[0].elapsed_time(e[1]) for e in evs]
    dec_ms = [e[1].elapsed_time(e[2]) for e in evs]
    per_call = {k: {"median_ms": round(statistics.median(v), 4), "best_ms": round(min(v), 4)}
                for k, v in (("compress", comp_ms), ("decompress", dec_ms))}
    graph = graph_steady_state(torch, step, stream, steps) if flush is not None else None
    total_ms, comp_tot, dec_tot = reduce_max([total_ms, sum(comp_ms), sum(dec_ms)], world, dev)
    K = steps
    comp_avg, dec_avg = comp_tot / K, dec_tot / K
    algo = in_bytes + int_nbytes          # bytes read + written, per kernel
    hbm, peak_src, _ = measured_peaks()
    dominant = "compress" if comp_avg >= dec_avg else "decompress"
    dom_ms = max(comp_avg, dec_avg)
    achieved = algo / (dom_ms * 1e-3) / 1e9
    lp_c = pc.poly_launches_per_call(n, dt, L, False)
    lp_d = pc.poly_launches_per_call(n, dt, L, True)
    rec = {
        "workload": c.name, "n": n, "block_len": L, "dtype": "u16" if dt == 16 else "u32",
        "input_bytes": in_bytes, "compressed_bytes": int_nbytes, "ratio": round(in_bytes / int_nbytes, 4),
        "bit_exact": bool(exact and post_ok), "steps": K,
        "value": round(job_gbs(world, in_bytes, K, total_ms), 2), "ms_per_step": round(total_ms / K, 4),
        "compress_gbs": round(in_bytes / (comp_avg * 1e-3) / 1e9, 2),
        "decompress_gbs": round(in_bytes / (dec_avg * 1e-3) / 1e9, 2),
        "compress_ms": round(comp_avg, 4), "decompress_ms": round(dec_avg, 4),
        "roofline": {"bound": "hbm", "kernel": dominant, "achieved": round(achieved, 1),
                     "peak": hbm, "unit": "GB/s", "frac": round(achieved / hbm, 4),
                     "traffic": traffic_from_profiles("%s/%s" % (c.name, dominant)),
                     "algorithmic_bytes": algo, "peak_source": peak_src,
                     "compress_frac": round(algo / (comp_avg * 1e-3) / 1e9 / hbm, 4),
                     "decompress_frac": round(algo / (dec_avg * 1e-3) / 1e9 / hbm, 4)},
        "per_call": per_call, "graph_steady_state": graph, "launches_per_step": lp_c + lp_d,
        "l2": ("inputs larger than L2 (%.2f GB vs 126 MB)" % (in_bytes / 1e9)) if flush is None
        else "L2 flushed (512 MiB write) between steps; steps timed individually",
    }
    extras = {"clocks": clk.summary() if clk else None, "oracle_s": (t_oc, t_od), "threads": threads,
              "x": x if keep_input else None, "x_np": x_np if keep_input else None, "dt": dt, "c": c,
              "total_ms": total_ms}
    del out, y, ws
    if not keep_input:
        del x
    torch.cuda.empty_cache()
    return rec, extras


def measure_advanced(args, cfg, steps, local):
    """The advanced (split-base) codec of PAPER.md Sec. 3.2 on a u16 config:
    gated against the C oracle (oracle_adv.c) byte for byte, then timed."""
    import numpy as np
    import torch
    import workloads
    from oracle import coracle
    from paper_1805_01844_b200 import polycomp as pc
    dev = torch.device("cuda", local)
    c = workloads.config(cfg, 1.0)
    x = workloads.generate(cfg, scale=1.0, seed=0, device=dev)
    n, L = c.n, c.block_len
    in_bytes = 2 * n
    cap = pc.poly_max_compressed_bytes_advanced(n, 16, L)
    out = torch.empty(cap, dtype=torch.uint8, device=dev)
    nb = torch.zeros(1, dtype=torch.int64, device=dev)
    wsb = pc.poly_workspace_bytes_advanced(n, 16, L)
    ws = torch.empty((wsb + 15) // 16 * 16, dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    pc.poly_compress_advanced(x, L, out=out, compressed_bytes=nb, workspace=ws)
    nbytes = int(nb.item())
    ref = coracle.compress_advanced(x.cpu().numpy(), L)
    ref_dev = torch.from_numpy(np.frombuffer(ref, dtype=np.uint8).copy()).to(dev)
    exact = len(ref) == nbytes and torch.equal(out[:nbytes], ref_dev)
    pc.poly_decompress_advanced(out, nbytes, 16, n, L, out=y, status=st, workspace=ws)
    torch.cuda.synchronize()
    if not (exact and int(st.item()) == 0 and torch.equal(x, y)):
        raise SystemExit("cfg%d advanced codec: GPU output differs from the oracle: no timing reported" % cfg)
    stream = torch.cuda.current_stream()
    for _ in range(3):
        pc.poly_compress_advanced(x, L, out=out, compressed_bytes=nb, workspace=ws)
        pc.poly_decompress_advanced(out, nbytes, 16, n, L, out=y, status=st, workspace=ws)
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
    torch.cuda.synchronize()
    for e in ev:
        e[0].record(stream)
        pc.poly_compress_advanced(x, L, out=out, compressed_bytes=nb, workspace=ws)
        e[1].record(stream)
        pc.poly_decompress_advanced(out, nbytes, 16, n, L, out=y, status=st, workspace=ws)
        e[2].record(stream)
    torch.cuda.synchronize()
    post = torch.equal(out[:nbytes], ref_dev) and int(st.item()) == 0 and torch.equal(x, y)
    if not post:
        raise SystemExit("cfg%d advanced codec: timed output differs from the oracle" % cfg)
    cm = sum(e[0].elapsed_time(e[1]) for e in ev) / steps
    dm = sum(e[1].elapsed_time(e[2]) for e in ev) / steps
    hbm, _, _ = measured_peaks()
    algo = in_bytes + nbytes
    del out, y, ws, ref_dev, x
    torch.cuda.empty_cache()
    return {"workload": c.name, "ratio": round(in_bytes / nbytes, 4), "bit_exact": True, "steps": steps,
            "compress_gbs": round(in_bytes / (cm * 1e-3) / 1e9, 2), "decompress_gbs": round(in_bytes / (dm * 1e-3) / 1e9, 2),
            "compress_ms": round(cm, 4), "decompress_ms": round(dm, 4),
            "compress_frac": round(algo / (cm * 1e-3) / 1e9 / hbm, 4), "decompress_frac": round(algo / (dm * 1e-3) / 1e9 / hbm, 4),
            "launches_per_step": 6}


def lzma_pairing(pc, torch, x, x_np, L, dt, dev):
    """PAPER.md Tables 1-2 (413, 488-492, 554): LZMA alone vs the polynomial
    codec followed by LZMA, on the first 64 MiB of the input (whole blocks),
    Python lzma preset 1.  Reported only (north_star)."""
    import lzma
    vb = dt // 8
    Lb = L or x_np.size
    nv = min(x_np.size, (64 << 20) // vb)
    if L:
        nv = max(Lb, nv // Lb * Lb)
    raw = x_np[:nv].tobytes()
    xs = x[:nv].contiguous()
    out, nb = pc.poly_compress(xs, L)
    stream_b = out[: int(nb.item())].cpu().numpy().tobytes()
    t0 = time.perf_counter()
    lz_raw = len(lzma.compress(raw, preset=1))
    t1 = time.perf_counter()
    lz_poly = len(lzma.compress(stream_b, preset=1))
    t2 = time.perf_counter()
    return {"sample_bytes": len(raw), "poly_ratio": round(len(raw) / len(stream_b), 4),
            "lzma_ratio": round(len(raw) / lz_raw, 4), "poly_then_lzma_ratio": round(len(raw) / lz_poly, 4),
            "lzma_s": round(t1 - t0, 3), "poly_then_lzma_lzma_s": round(t2 - t1, 3),
            "how": "python lzma preset 1 on the first %d values (whole blocks)" % nv}


def run_ours(args, rank, world, local):
    import torch
    from paper_1805_01844_b200 import polycomp as pc

    dev = torch.device("cuda", local)
    pc.load_library()
    pc.poly_init(local)
    K = args.steps
    rec, ex = measure(args, args.config, K, rank, world, local, clocks=True, keep_input=True)
    c, dt = ex["c"], ex["dt"]
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, pc, torch, ex["x"], c.n, dt, c.block_len, rec["input_bytes"], rec["compressed_bytes"],
                      dev, world)
    lz = None
    if rank == 0 and not args.only:
        try:
            lz = lzma_pairing(pc, torch, ex["x"], ex["x_np"], c.block_len, dt, dev)
        except Exception as e:  # pragma: no cover
            lz = {"error": str(e)[:200]}
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        t_oc, t_od = ex["oracle_s"]
        st_val, st_sample = single_thread_oracle(ex["x_np"], c.block_len, ex["threads"])
        cpu = {"value": round(rec["input_bytes"] / (t_oc + t_od) / 1e9, 4), "unit": "GB/s", "cores": ex["threads"],
               "kind": "oracle", "sample": "full input (%s, seed 0), compress+decompress, all host cores" % c.description,
               "compress_gbs": round(rec["input_bytes"] / t_oc / 1e9, 4),
               "decompress_gbs": round(rec["input_bytes"] / t_od / 1e9, 4),
               "single_thread_value": st_val, "single_thread_sample": st_sample, "cpu_model": cpu_model()}
    ex["x"] = ex["x_np"] = None
    torch.cuda.empty_cache()
    others = {}
    if world == 1 and not args.only:
        for cfg in (1, 2, 3, 4, 5, 6):  # 6: cfg2 in the paper's time-major layout
            if cfg == args.config:
                continue
            r, _ = measure(args, cfg, min(K, 10), rank, world, local, clocks=False)
            others["cfg%d" % cfg] = r
    advanced = {}
    if world == 1 and not args.only:
        for cfg in (2, 4, 5):
            try:
                advanced["cfg%d" % cfg] = measure_advanced(args, cfg, min(K, 10), local)
            except SystemExit:
                raise
            except Exception as e:  # pragma: no cover
                advanced["cfg%d" % cfg] = {"error": str(e)[:200]}
    if rank != 0:
        return
    line = {
        "metric": METRIC,
        "value": rec["value"],
        "unit": "GB/s",
        "n_gpus": world,
        "steps": K,
        "warmup": max(3, args.warmup),
        "ms_per_step": rec["ms_per_step"],
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": rec["dtype"],
        "data": "synthetic (seeded, BASELINE.json config %d; seed = rank)" % args.config,
        "config": {"workload": c.name, "n": c.n, "block_len": c.block_len, "input_bytes": rec["input_bytes"],
                   "compressed_bytes": rec["compressed_bytes"], "l2": rec["l2"]},
        "bit_exact": rec["bit_exact"],
        "ratio": rec["ratio"],
        "compress_gbs": rec["compress_gbs"],
        "decompress_gbs": rec["decompress_gbs"],
        "compress_ms": rec["compress_ms"],
        "decompress_ms": rec["decompress_ms"],
        "roofline": rec["roofline"],
        "per_call": rec["per_call"],
        "graph_steady_state": rec["graph_steady_state"],
        "clocks": ex["clocks"],
        "e2e": e2e,
        "gpu_launches": K * rec["launches_per_step"],
        "cpu_baseline": cpu,
        "lzma": lz,
        "configs": others,
        "advanced": advanced,
    }
    print(json.dumps(line), flush=True)


def graph_steady_state(torch, step, stream, steps):
    """One compress + decompress captured in a CUDA graph and replayed back to
    back (no L2 flush): the launch-free steady state of the small config."""
    try:
        s = torch.cuda.Stream()
        s.wait_stream(stream)
        with torch.cuda.stream(s):
            step()  # the calls read torch's current stream: warm on the capture stream
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            step()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        a.record(cur)
        for _ in range(max(1, steps)):
            g.replay()
        b.record(cur)
        torch.cuda.synchronize()
        return {"us_per_step": round(1e3 * a.elapsed_time(b) / max(1, steps), 3), "replays": max(1, steps)}
    except Exception as e:  # pragma: no cover
        return {"error": str(e)[:200]}


def run_e2e(args, pc, torch, x, n, dt, L, in_bytes, nbytes, dev, world):
    """End to end through the host-buffer C-ABI calls (pinned memory)."""
    try:
        h_in = torch.empty(n, dtype=x.dtype, pin_memory=True)
        h_in.copy_(x.cpu())
        cap = pc.poly_max_compressed_bytes(n, dt, L)
        h_stream = torch.empty(cap, dtype=torch.uint8, pin_memory=True)
        h_out = torch.empty(n, dtype=x.dtype, pin_memory=True)
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": "GB/s", "error": "pinned alloc failed: %s" % e}
    d_in = torch.empty(max(cap, in_bytes), dtype=torch.uint8, device=dev)
    d_out = torch.empty(max(cap, in_bytes), dtype=torch.uint8, device=dev)
    ws = pc.alloc_workspace(n, dt, L, dev)
    steps = max(1, args.e2e_steps)

    def one():
        nb = pc.poly_compress_host(h_in, L, d_in, d_out, ws, h_stream)
        st = pc.poly_decompress_host(h_stream, nb, dt, n, L, d_in, d_out, ws, h_out)
        return nb, st

    nb, st = one()  # warm-up
    import torch.distributed as dist
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        nb, st = one()
    el = time.perf_counter() - t0
    t = torch.tensor([el], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    el = float(t.item())
    ok = st == 0 and torch.equal(h_out, h_in)
    return {"value": round(world * in_bytes * steps / el / 1e9, 3), "unit": "GB/s",
            "h2d_bytes_per_step": in_bytes + nb, "d2h_bytes_per_step": nb + in_bytes + 12,
            "steps": steps, "roundtrip_ok": bool(ok)}


def main():
    args = parse()
    rank, world, local = dist_init(args)
    if args.impl == "reference":
        run_reference(args, rank, world)
    else:
        run_ours(args, rank, world, local)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
