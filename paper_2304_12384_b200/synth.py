"""Seeded synthetic frame generators for the five BASELINE.json configs.

This module holds input generation only -- none of the method's arithmetic
(no transform, no features).  It is the one module both the CUDA path and
the CPU oracle consume: every parity test generates bytes here once and
feeds the same bytes to both sides.

The generators stand in for the paper's unnamed "UHD 8-bit videos"
and the VCD dataset, neither of which is available.  Recipes
(BASELINE.json ``configs``; readings in DESIGN.md "Input recipe"):

* config 1 (CIF, seed 0): clamp(rint(128 + 60 sin(2 pi (x cos a + y sin a)/L
  + 0.3 t) + N(0, 8^2)), 0, 255); Y: a = 0.7 rad, L = 24 px; U/V: a = 1.1,
  L = 12 at half resolution.
* generator G(seed) (configs 2-5): per plane, 3 oriented sinusoids
  (theta ~ U[0, pi), lambda ~ U[4, 64] px, A ~ U[10, 40], phi ~ U[0, 2 pi),
  v ~ U[0, 4] px/frame along the wave normal) plus Gaussian noise sigma ~
  U[4, 12]; frame 0 is a scene cut and every later frame cuts with
  probability 0.1, redrawing all parameters.  Config 4 samples are
  clamp(rint(4 * value), 0, 1023) stored as uint16.

Structure parameters come from a numpy PCG64 stream that is replayed from
frame 0 (cheap); the pixel field and noise are computed with torch on the
requested device, noise seeded per (seed, t, plane) so any frame -- e.g. a
rank's halo frame -- can be generated on its own.  CPU and CUDA noise
streams differ, so bytes depend on the device; parity always compares both
sides on the same bytes.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch


@dataclass(frozen=True)
class Config:
    name: str
    width: int
    height: int
    bit_depth: int
    block_size: int
    lowpass: bool
    n_frames: int
    seed: int


CONFIGS = {
    1: Config("cif_8bit_full32", 352, 288, 8, 32, False, 16, 0),
    2: Config("1080p_8bit_full32", 1920, 1080, 8, 32, False, 240, 1),
    3: Config("uhd_8bit_lowpass32", 3840, 2160, 8, 32, True, 600, 2),
    4: Config("uhd_10bit_full16", 3840, 2160, 10, 16, False, 600, 3),
    5: Config("uhd_8bit_lowpass32_x4800", 3840, 2160, 8, 32, True, 4800, 10),
}
SEGMENT_FRAMES = 600  # config 5: 8 segments of 600 frames, seeds 10..17


def _noise(shape, seed_words, device):
    s = int(np.random.SeedSequence(list(seed_words)).generate_state(1, np.uint64)[0] & ((1 << 63) - 1))
    g = torch.Generator(device=device)
    g.manual_seed(s)
    return torch.randn(shape, generator=g, device=device, dtype=torch.float64)


def _grid(h, w, device):
    y = torch.arange(h, device=device, dtype=torch.float64).view(h, 1)
    x = torch.arange(w, device=device, dtype=torch.float64).view(1, w)
    return x, y


def cif_frames(n_frames: int = 16, device="cpu", width: int = 352, height: int = 288, seed: int = 0):
    """Config 1 frames -> (Y, U, V) uint8 tensors [F][H][W], [F][H/2][W/2]."""
    out = []
    for p, (w, h, a, L) in enumerate(((width, height, 0.7, 24.0), (width // 2, height // 2, 1.1, 12.0),
                                      (width // 2, height // 2, 1.1, 12.0))):
        x, y = _grid(h, w, device)
        base = 2.0 * math.pi * (x * math.cos(a) + y * math.sin(a)) / L
        frames = torch.empty((n_frames, h, w), dtype=torch.uint8, device=device)
        for t in range(n_frames):
            v = 128.0 + 60.0 * torch.sin(base + 0.3 * t) + 8.0 * _noise((h, w), (seed, t, p), device)
            frames[t] = torch.clamp(torch.round(v), 0, 255).to(torch.uint8)
        out.append(frames)
    return tuple(out)


def _structure(seed: int, n_frames: int):
    """Replay G(seed)'s structure stream: per frame, the parameters in force
    (cut frame t_s and per-plane sinusoid/sigma parameters)."""
    rng = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, 0])))
    params = []
    cur = None
    for t in range(n_frames):
        cut = (t == 0) or (rng.random() < 0.1)
        if cut:
            planes = []
            for _p in range(3):
                sines = []
                for _s in range(3):
                    theta = rng.uniform(0.0, math.pi)
                    lam = rng.uniform(4.0, 64.0)
                    A = rng.uniform(10.0, 40.0)
                    phi = rng.uniform(0.0, 2.0 * math.pi)
                    v = rng.uniform(0.0, 4.0)
                    sines.append((theta, lam, A, phi, v))
                sigma = rng.uniform(4.0, 12.0)
                planes.append((sines, sigma))
            cur = (t, planes)
        params.append(cur)
    return params


def g_frames(seed: int, width: int, height: int, n_frames: int, bit_depth: int = 8, first_t: int = 0,
             device="cpu", out=None):
    """Frames first_t .. first_t+n_frames-1 of G(seed) -> (Y, U, V) tensors.

    8-bit: uint8; 10-bit: uint16 holding clamp(rint(4 value), 0, 1023).
    ``out`` may pass preallocated (Y, U, V) tensors to fill."""
    params = _structure(seed, first_t + n_frames)
    dims = ((width, height), (width // 2, height // 2), (width // 2, height // 2))
    dt = torch.uint8 if bit_depth == 8 else torch.int16  # int16 storage == LE uint16 for 0..1023
    if out is None:
        out = tuple(torch.empty((n_frames, h, w), dtype=dt, device=device) for (w, h) in dims)
    hi = 255 if bit_depth == 8 else 1023
    scale = 1.0 if bit_depth == 8 else 4.0
    grids = [_grid(h, w, device) for (w, h) in dims]
    for i in range(n_frames):
        t = first_t + i
        ts, planes = params[t]
        for p in range(3):
            x, y = grids[p]
            w, h = dims[p]
            sines, sigma = planes[p]
            v = torch.full((h, w), 128.0, dtype=torch.float64, device=device)
            for (theta, lam, A, phi, vel) in sines:
                # angle addition keeps this an outer sum: sin(ax + by + c)
                arg_x = x * (2.0 * math.pi * math.cos(theta) / lam)
                arg_y = y * (2.0 * math.pi * math.sin(theta) / lam) + (phi - 2.0 * math.pi * vel * (t - ts) / lam)
                v += A * torch.sin(arg_x + arg_y)
            v += sigma * _noise((h, w), (seed, 1, t, p), device)
            q = torch.clamp(torch.round(v * scale), 0, hi)
            out[p][i] = q.to(dt)
    return out


def config_frames(cfg_id: int, device="cpu", n_frames: int | None = None, first_t: int = 0,
                  width: int | None = None, height: int | None = None):
    """Frames of BASELINE.json config ``cfg_id`` (optionally fewer frames or a
    smaller geometry for tests).  Config 5 frames are indexed by global POC
    across its 8 segments."""
    c = CONFIGS[cfg_id]
    W = width or c.width
    H = height or c.height
    F = c.n_frames if n_frames is None else n_frames
    if cfg_id == 1:
        assert first_t == 0
        return cif_frames(F, device, W, H, c.seed)
    if cfg_id != 5:
        return g_frames(c.seed, W, H, F, c.bit_depth, first_t, device)
    dt = torch.uint8
    out = tuple(torch.empty((F, h, w), dtype=dt, device=device) for (w, h) in ((W, H), (W // 2, H // 2),
                                                                               (W // 2, H // 2)))
    i = 0
    while i < F:
        poc = first_t + i
        seg, t0 = divmod(poc, SEGMENT_FRAMES)
        m = min(F - i, SEGMENT_FRAMES - t0)
        g_frames(c.seed + seg, W, H, m, 8, t0, device, out=tuple(o[i:i + m] for o in out))
        i += m
    return out


def as_numpy_planes(Y, U, V):
    """torch planes -> numpy arrays with the oracle's dtypes (uint8 / uint16)."""
    res = []
    for p in (Y, U, V):
        a = p.detach().cpu().numpy()
        if a.dtype == np.int16:
            a = a.view(np.uint16)
        res.append(a)
    return tuple(res)


def with_pitch(planes, align: int = 16):
    """Copy [F][H][W] planes into buffers whose row pitch is rounded up to
    ``align`` bytes (libvca requires 16-byte aligned pitches), returning
    strided views of the same shape."""
    res = []
    for p in planes:
        F, H, W = p.shape
        es = p.element_size()
        wp = ((W * es + align - 1) // align * align) // es
        buf = torch.zeros((F, H, wp), dtype=p.dtype, device=p.device)
        buf[:, :, :W] = p
        res.append(buf[:, :, :W])
    return tuple(res)
