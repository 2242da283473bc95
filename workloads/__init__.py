"""Seeded synthetic inputs for the five BASELINE.json configurations.

This module only draws random numbers and lays them out; it holds none of the
codec's arithmetic (no min/max, base, capacity, packing), so both the oracle
(tests, bench cpu_baseline) and the CUDA path read the same bytes from it.

Recipes:
  cfg1  1,048,576 u16, clip(round(N(300, 5^2)), 0, 65535), one block (L = 0).
  cfg2  [events][1855 pixels][30 samples] u16, pixel-major, L = 30: pedestal
        noise N(250, 4^2); with probability 0.02 per (event, pixel) a pulse
        A*exp(-(t-t0)^2 / (2*3^2)), t0 ~ U{5..25}, A ~ Exp(mean 200);
        value = clip(round(pedestal + pulse), 0, 65535).  Stands in for the CTA
        PROD_3 waveform files, which are absent.
  cfg3  2^28 u32, L = 65,536: block i draws b_i = floor(2^U(1,20)) and
        uniform integers in [0, b_i) (float64 floor(u*b), clamped).
  cfg4  2^29 u16, clip(round(N(2000, 50^2))), each value replaced by 4095 with
        probability 1e-4, L = 1,024.
  cfg5  2^31 u16, L = 4,096; block i mod 3: 0 -> Poisson(20),
        1 -> round(N(1000, 30^2)), 2 -> uniform integers [0, 15].
  cfg6  cfg2's values in the paper's time-major matrix layout M_{i,j}
        ("M_{i,j} corresponds to the i-th time"): per
        event a [30 time samples][1855 pixels] matrix, row-major, one block
        per time row (L = 1855) -- SURVEY.md Sec. 8(f) row 4.
`scale` < 1 shrinks the number of events / blocks / values while keeping the
distribution, the block length and the layout (used by the CPU-sized tests).
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

CHUNK = 1 << 25


@dataclass(frozen=True)
class Config:
    name: str
    dtype: torch.dtype
    n: int
    block_len: int
    description: str


CTA_PIXELS = 1855
CTA_SAMPLES = 30
CTA_EVENTS = 10_000


def config(cfg: int, scale: float = 1.0) -> Config:
    """Return the (possibly scaled) shape of BASELINE config `cfg` (1..5)."""
    if cfg == 1:
        return Config("cfg1_gauss_single_block", torch.uint16, max(1, int((1 << 20) * scale)), 0,
                      "1,048,576 u16 round(N(300,5^2)), one block")
    if cfg == 2:
        ev = max(1, int(CTA_EVENTS * scale))
        return Config("cfg2_cta_camera_events", torch.uint16, ev * CTA_PIXELS * CTA_SAMPLES, CTA_SAMPLES,
                      "%d events x 1855 pixels x 30 samples u16, L=30" % ev)
    if cfg == 3:
        nb = max(1, int(4096 * scale))
        return Config("cfg3_uniform_u32_logbase", torch.uint32, nb * 65536, 65536,
                      "%d blocks x 65536 u32, b_i log-uniform 2..2^20" % nb)
    if cfg == 4:
        return Config("cfg4_gauss_outliers_u16", torch.uint16, max(1024, int((1 << 29) * scale)), 1024,
                      "u16 round(N(2000,50^2)) + 1e-4 outliers at 4095, L=1024")
    if cfg == 5:
        n = max(4096 * 3, int((1 << 31) * scale))
        return Config("cfg5_mixed_blocks_u16", torch.uint16, n, 4096,
                      "u16 L=4096 cycling Poisson(20) / N(1000,30^2) / U[0,15]")
    if cfg == 6:
        ev = max(1, int(CTA_EVENTS * scale))
        return Config("cfg6_cta_time_major", torch.uint16, ev * CTA_PIXELS * CTA_SAMPLES, CTA_PIXELS,
                      "%d events x 30 samples x 1855 pixels u16 (time-major M_ij), L=1855" % ev)
    raise ValueError("cfg must be 1..6")


def _gen(device, seed):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def _to_u16(x_f: torch.Tensor) -> torch.Tensor:
    return torch.clamp(torch.round(x_f), 0, 65535).to(torch.int32).to(torch.uint16)


def generate(cfg: int, scale: float = 1.0, seed: int = 0, device="cpu") -> torch.Tensor:
    """Seeded synthetic input for config `cfg` on `device` (1-D, u16 or u32)."""
    c = config(cfg, scale)
    g = _gen(device, seed)
    if cfg == 1:
        x = torch.randn(c.n, generator=g, device=device, dtype=torch.float32) * 5.0 + 300.0
        return _to_u16(x)
    if cfg == 2:
        ev = c.n // (CTA_PIXELS * CTA_SAMPLES)
        out = torch.empty(c.n, dtype=torch.uint16, device=device)
        t = torch.arange(CTA_SAMPLES, device=device, dtype=torch.float32)
        ev_chunk = max(1, CHUNK // (CTA_PIXELS * CTA_SAMPLES))
        for e0 in range(0, ev, ev_chunk):
            e1 = min(ev, e0 + ev_chunk)
            shape = (e1 - e0, CTA_PIXELS)
            ped = torch.randn(shape + (CTA_SAMPLES,), generator=g, device=device) * 4.0 + 250.0
            pulsed = torch.rand(shape, generator=g, device=device) < 0.02
            t0 = torch.randint(5, 26, shape, generator=g, device=device).to(torch.float32)
            amp = torch.empty(shape, device=device).exponential_(1.0 / 200.0, generator=g)
            pulse = amp[..., None] * torch.exp(-((t - t0[..., None]) ** 2) / (2.0 * 3.0 ** 2))
            val = ped + torch.where(pulsed[..., None], pulse, torch.zeros_like(pulse))
            out[e0 * CTA_PIXELS * CTA_SAMPLES: e1 * CTA_PIXELS * CTA_SAMPLES] = _to_u16(val).reshape(-1)
        return out
    if cfg == 3:
        nb = c.n // 65536
        out = torch.empty(c.n, dtype=torch.int64, device=device)
        u = torch.rand(nb, generator=g, device=device, dtype=torch.float64) * 19.0 + 1.0
        b = torch.floor(torch.pow(2.0, u)).to(torch.int64)
        per = max(1, CHUNK // 65536)
        for b0 in range(0, nb, per):
            b1 = min(nb, b0 + per)
            r = torch.rand((b1 - b0, 65536), generator=g, device=device, dtype=torch.float64)
            bb = b[b0:b1, None]
            v = torch.minimum(torch.floor(r * bb.to(torch.float64)).to(torch.int64), bb - 1)
            out[b0 * 65536: b1 * 65536] = v.reshape(-1)
        return out.to(torch.uint32)
    if cfg == 4:
        out = torch.empty(c.n, dtype=torch.uint16, device=device)
        for i0 in range(0, c.n, CHUNK):
            i1 = min(c.n, i0 + CHUNK)
            x = torch.randn(i1 - i0, generator=g, device=device) * 50.0 + 2000.0
            outl = torch.rand(i1 - i0, generator=g, device=device) < 1e-4
            x = torch.where(outl, torch.full_like(x, 4095.0), x)
            out[i0:i1] = _to_u16(x)
        return out
    if cfg == 5:
        L = 4096
        nb = (c.n + L - 1) // L
        out = torch.empty(c.n, dtype=torch.uint16, device=device)
        per = max(3, (CHUNK // L) // 3 * 3)
        for b0 in range(0, nb, per):
            b1 = min(nb, b0 + per)
            nblk = b1 - b0
            kind = (torch.arange(b0, b1, device=device) % 3)[:, None]
            lam = torch.full((nblk, L), 20.0, device=device)
            pois = torch.poisson(lam, generator=g)
            gau = torch.randn((nblk, L), generator=g, device=device) * 30.0 + 1000.0
            uni = torch.randint(0, 16, (nblk, L), generator=g, device=device).to(torch.float32)
            v = torch.where(kind == 0, pois, torch.where(kind == 1, gau, uni))
            flat = _to_u16(v).reshape(-1)
            lo = b0 * L
            hi = min(c.n, b1 * L)
            out[lo:hi] = flat[: hi - lo]
        return out
    if cfg == 6:  # cfg2's values, each event's [pixel][time] matrix transposed to [time][pixel]
        x = generate(2, scale=scale, seed=seed, device=device)
        ev = c.n // (CTA_PIXELS * CTA_SAMPLES)
        out = torch.empty_like(x)
        per = max(1, CHUNK // (CTA_PIXELS * CTA_SAMPLES))
        for e0 in range(0, ev, per):
            e1 = min(ev, e0 + per)
            blk = x[e0 * CTA_PIXELS * CTA_SAMPLES: e1 * CTA_PIXELS * CTA_SAMPLES].view(torch.int16)
            blk = blk.view(e1 - e0, CTA_PIXELS, CTA_SAMPLES).transpose(1, 2).contiguous().view(-1)
            out.view(torch.int16)[e0 * CTA_PIXELS * CTA_SAMPLES: e1 * CTA_PIXELS * CTA_SAMPLES] = blk
        return out
    raise ValueError(cfg)
