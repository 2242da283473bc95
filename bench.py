#!/usr/bin/env python
"""Benchmark of the B200 polynomial-codec hot path (one JSON line on rank 0).

A step = one pass of the whole hot path over one batch: poly_compress then
poly_decompress of the BASELINE workload (default cfg2, the CTA-like camera
events, 1.113 GB of u16; BASELINE.json configs[1]), inputs resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

value     = uncompressed bytes of all ranks x K / max-over-ranks device time of
            the K steps (GB/s, compress + decompress in series).
e2e       = the same metric through poly_compress_host / poly_decompress_host
            (pinned host buffers, H2D + D2H inside the timed region).
roofline  = the dominant kernel's algorithmic bytes (I + C, read + written)
            per launch / its CUDA-event duration, against MEASURED_PEAKS.json.
cpu_baseline = the C oracle (oracle/oracle.c, all host cores) on a bounded
            sample of the same workload (rank 0, N = 1 only).
--impl reference times that oracle as the reference arm.
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
    p.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--e2e-steps", type=int, default=3)
    p.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU work for the oracle sample")
    p.add_argument("--verify", action="store_true", help="check the stream against the oracle first")
    p.add_argument("--no-roundtrip-check", action="store_true",
                   help="timing experiments (POLY_DEBUG) only: skip the round-trip check")
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


def oracle_sample(cfg: int, target_seconds: float):
    """A bounded sample of the workload for the CPU oracle: whole blocks from
    the start of the same seeded input (generated on the CPU at that size)."""
    import workloads
    full = workloads.config(cfg, 1.0)
    # rough oracle speed ~ 0.25 GB/s/core-equivalent for compress+decompress
    frac = {1: 1.0, 2: 0.01, 3: 1 / 64, 4: 1 / 64, 5: 1 / 256}[cfg]
    scale = frac * max(0.25, min(4.0, target_seconds / 12.0))
    scale = min(scale, 1.0)
    c = workloads.config(cfg, scale)
    x = workloads.generate(cfg, scale=scale, seed=0, device="cpu").numpy()
    return x, c, "first %d of %d values (%s, seed 0, generated on the host)" % (c.n, full.n, c.description)


def time_oracle(cfg: int, target_seconds: float, steps: int = 1):
    from oracle import coracle
    import numpy as np
    x, c, sample = oracle_sample(cfg, target_seconds)
    threads = coracle.default_threads()
    times = []
    for _ in range(max(1, steps)):
        t0 = time.perf_counter()
        s = coracle.compress(x, c.block_len, threads=threads)
        y, st = coracle.decompress(s, threads=threads)
        times.append(time.perf_counter() - t0)
        assert st == 0 and np.array_equal(y, x)
    gbs = x.nbytes / (sum(times) / len(times)) / 1e9
    # one thread on the first 1/threads of the sample's blocks (same per-thread work)
    L = c.block_len or x.size
    n1 = max(L, (x.size // max(1, threads)) // L * L) if c.block_len else x.size
    x1 = x[:n1]
    t0 = time.perf_counter()
    s1 = coracle.compress(x1, c.block_len, threads=1)
    y1, st1 = coracle.decompress(s1, threads=1)
    t1 = time.perf_counter() - t0
    assert st1 == 0 and np.array_equal(y1, x1)
    return {"value": round(gbs, 4), "unit": "GB/s", "cores": threads, "kind": "oracle",
            "sample": sample + "; compress+decompress, all host cores",
            "single_thread_value": round(x1.nbytes / t1 / 1e9, 4),
            "single_thread_sample": "first %d values, 1 thread" % n1,
            "cpu_model": cpu_model()}, times, x.nbytes


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
    if rank != 0:
        return
    import workloads
    c = workloads.config(args.config, 1.0)
    for _ in range(args.warmup if args.warmup <= 1 else 1):
        pass
    cb, times, nbytes = time_oracle(args.config, args.cpu_seconds / 2, steps=max(1, args.steps))
    tot = sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": cb["value"], "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * tot / len(times), 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u16" if c.dtype.itemsize == 2 else "u32",
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


def run_ours(args, rank, world, local):
    import torch
    import workloads
    from paper_1805_01844_b200 import polycomp as pc

    dev = torch.device("cuda", local)
    pc.load_library()
    pc.poly_init(local)
    c = workloads.config(args.config, 1.0)
    dt = 16 if c.dtype == torch.uint16 else 32
    x = workloads.generate(args.config, scale=1.0, seed=rank, device=dev)
    n, L = c.n, c.block_len
    in_bytes = n * (dt // 8)
    cap = pc.poly_max_compressed_bytes(n, dt, L)
    out = torch.empty(cap, dtype=torch.uint8, device=dev)
    nb = torch.zeros(1, dtype=torch.int64, device=dev)
    ws = pc.alloc_workspace(n, dt, L, dev)
    y = torch.empty_like(x)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    stream = torch.cuda.current_stream()
    flush = None
    if in_bytes < 256 << 20:
        flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)

    def step(ev=None):
        if ev is not None:
            ev[0].record(stream)
        pc.poly_compress(x, L, out=out, compressed_bytes=nb, workspace=ws)
        if ev is not None:
            ev[1].record(stream)
        pc.poly_decompress(out, int_nbytes, dt, n, L, out=y, status=st, workspace=ws)
        if ev is not None:
            ev[2].record(stream)

    # sizes are needed on the host for decompress: one untimed compress
    pc.poly_compress(x, L, out=out, compressed_bytes=nb, workspace=ws)
    int_nbytes = int(nb.item())
    pc.poly_decompress(out, int_nbytes, dt, n, L, out=y, status=st, workspace=ws)
    torch.cuda.synchronize()
    ok = int(st.item()) == 0 and torch.equal(x, y)
    if not ok and not args.no_roundtrip_check:
        raise SystemExit("round trip failed on rank %d (status %d)" % (rank, int(st.item())))
    if args.verify and rank == 0:
        from oracle import coracle
        ref = coracle.compress(x.cpu().numpy(), L)
        if out[:int_nbytes].cpu().numpy().tobytes() != ref:
            raise SystemExit("stream differs from the oracle")

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    import torch.distributed as dist
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        if flush is None:
            t_start.record(stream)
            for i in range(args.steps):
                step(evs[i])
            t_end.record(stream)
            torch.cuda.synchronize()
            total_ms = t_start.elapsed_time(t_end)
        else:  # small input (cfg1): flush L2 between steps, time the steps only
            for i in range(args.steps):
                flush.fill_(i & 0xff)
                step(evs[i])
            torch.cuda.synchronize()
            total_ms = sum(e[0].elapsed_time(e[2]) for e in evs)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    comp_ms = [e[0].elapsed_time(e[1]) for e in evs]
    dec_ms = [e[1].elapsed_time(e[2]) for e in evs]
    per_call = {k: {"median_ms": round(statistics.median(v), 4), "best_ms": round(min(v), 4)}
                for k, v in (("compress", comp_ms), ("decompress", dec_ms))}
    graph = None
    if flush is not None:  # cfg1 (L2-resident): CUDA-graph steady state of one step
        graph = graph_steady_state(torch, step, stream, args.steps)
    total_ms, comp_tot, dec_tot = reduce_max([total_ms, sum(comp_ms), sum(dec_ms)], world, dev)
    K = args.steps
    value = job_gbs(world, in_bytes, K, total_ms)
    comp_avg, dec_avg = comp_tot / K, dec_tot / K
    algo = in_bytes + int_nbytes          # bytes read + written, both kernels
    hbm, peak_src, _ = measured_peaks()
    dominant = "compress" if comp_avg >= dec_avg else "decompress"
    dom_ms = max(comp_avg, dec_avg)
    achieved = algo / (dom_ms * 1e-3) / 1e9
    lp_c = pc.poly_launches_per_call(n, dt, L, False)
    lp_d = pc.poly_launches_per_call(n, dt, L, True)
    kern_key = "%s/%s" % (c.name, dominant)
    traffic = traffic_from_profiles(kern_key)

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, pc, torch, x, n, dt, L, in_bytes, int_nbytes, dev, world)

    if rank != 0:
        return
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        try:
            cpu, _, _ = time_oracle(args.config, args.cpu_seconds)
        except Exception as e:  # pragma: no cover
            cpu = {"value": None, "unit": "GB/s", "cores": None, "kind": "oracle", "sample": "failed: %s" % e}
    line = {
        "metric": METRIC,
        "value": round(value, 2),
        "unit": "GB/s",
        "n_gpus": world,
        "steps": K,
        "warmup": max(3, args.warmup),
        "ms_per_step": round(total_ms / K, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u16" if dt == 16 else "u32",
        "data": "synthetic (seeded, BASELINE.json config %d; seed = rank)" % args.config,
        "config": {"workload": c.name, "n": n, "block_len": L, "input_bytes": in_bytes,
                   "compressed_bytes": int_nbytes,
                   "l2": ("inputs larger than L2 (%.2f GB vs 126 MB)" % (in_bytes / 1e9)) if flush is None
                   else "L2 flushed (512 MiB write) between steps; steps timed individually"},
        "ratio": round(in_bytes / int_nbytes, 4),
        "compress_gbs": round(in_bytes / (comp_avg * 1e-3) / 1e9, 2),
        "decompress_gbs": round(in_bytes / (dec_avg * 1e-3) / 1e9, 2),
        "compress_ms": round(comp_avg, 4),
        "decompress_ms": round(dec_avg, 4),
        "roofline": {"bound": "hbm", "kernel": dominant, "achieved": round(achieved, 1),
                     "peak": hbm, "unit": "GB/s", "frac": round(achieved / hbm, 4),
                     "traffic": traffic, "algorithmic_bytes": algo, "peak_source": peak_src,
                     "other_kernel_frac": round(algo / (min(comp_avg, dec_avg) * 1e-3) / 1e9 / hbm, 4)},
        "per_call": per_call,
        "graph_steady_state": graph,
        "clocks": clk.summary(),
        "e2e": e2e,
        "gpu_launches": K * (lp_c + lp_d),
        "cpu_baseline": cpu,
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
