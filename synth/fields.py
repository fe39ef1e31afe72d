"""Synthetic stand-ins for the paper's datasets (NYX, ATM, Hurricane).

The real fields are not in the container; these generators reproduce their
shapes (ATM 1800x3600 and Hurricane 100x500x500; NYX 512^3 per
BASELINE.json) and the value-distribution features the paper names
(heavy-tailed density, fields with exact zeros, smooth vs hard fields,
PAPER.md:517-520, 545).  Recipes follow SURVEY.md section 8(d); DESIGN.md
section 4 restates them.

Every generator takes an explicit ``shape`` so tests can draw the same recipe
at small sizes.  Seeds: ``numpy.random.default_rng([config, field, sub])``.
Arithmetic is float64 internally and the result is cast to float32 at the end.
"""
from __future__ import annotations

import os

import numpy as np

try:  # multithreaded FFT when scipy is present (it is in this image)
    import scipy.fft as _fft

    def _rfftn(a):
        return _fft.rfftn(a, workers=os.cpu_count())

    def _irfftn(a, s):
        return _fft.irfftn(a, s=s, workers=os.cpu_count())
except Exception:  # pragma: no cover
    def _rfftn(a):
        return np.fft.rfftn(a)

    def _irfftn(a, s):
        return np.fft.irfftn(a, s=s)


CONFIGS = {
    1: dict(shape=(256, 256), n_fields=1, eb_rel=(1e-4,), strides=((1, 1),)),
    2: dict(shape=(1800, 3600), n_fields=100, eb_rel=(1e-4,), strides=((1, 1), (1, 10))),
    3: dict(shape=(100, 500, 500), n_fields=13, eb_rel=(1e-3, 1e-4, 1e-5), strides=((1, 1, 1),)),
    4: dict(shape=(512, 512, 512), n_fields=6, eb_rel=(1e-4,), strides=((1, 1, 1), (4, 4, 4))),
    5: dict(shape=(1024, 1024, 1024), n_fields=3,
            eb_rel=(1e-2, 1e-3, 1e-4, 1e-5, 1e-6, 1e-7), strides=((1, 1, 1),)),
}


def grf(shape, beta: float, rng: np.random.Generator) -> np.ndarray:
    """Gaussian random field with power spectrum |k|^-beta, mean 0, std 1 (float64).

    white N(0,1) -> rfftn -> multiply by |k|^(-beta/2) (k in cycles/cell, k=0
    term zeroed) -> irfftn -> standardise.  Periodic.
    """
    white = rng.standard_normal(shape)
    F = _rfftn(white)
    del white
    ks = [np.fft.fftfreq(n) for n in shape[:-1]] + [np.fft.rfftfreq(shape[-1])]
    k2 = np.zeros(F.shape, dtype=np.float64)
    for a, k in enumerate(ks):
        sh = [1] * len(shape)
        sh[a] = k.size
        k2 = k2 + (k.reshape(sh) ** 2)
    k2.flat[0] = 1.0
    amp = k2 ** (-beta / 4.0)
    amp.flat[0] = 0.0
    F *= amp
    del k2, amp
    g = _irfftn(F, s=shape)
    g -= g.mean()
    sd = g.std()
    return g / sd if sd > 0 else g


# --------------------------------------------------------------------------- C1
def c1_field(shape=(256, 256), seed: int = 0) -> np.ndarray:
    """Config 1: sum of 4 random sinusoids (wavelength 8-128 cells, A~U(0.5,2)) + N(0,1e-3^2)."""
    rng = np.random.default_rng(seed)
    y, x = np.meshgrid(np.arange(shape[0], dtype=np.float64),
                       np.arange(shape[1], dtype=np.float64), indexing="ij")
    f = np.zeros(shape, np.float64)
    for _ in range(4):
        A = rng.uniform(0.5, 2.0)
        lam = np.exp(rng.uniform(np.log(8.0), np.log(128.0)))
        th = rng.uniform(0.0, 2 * np.pi)
        ph = rng.uniform(0.0, 2 * np.pi)
        f += A * np.sin(2 * np.pi * (x * np.cos(th) + y * np.sin(th)) / lam + ph)
    f += rng.normal(0.0, 1e-3, size=shape)
    return f.astype(np.float32)


# --------------------------------------------------------------------------- C2
def c2_field(i: int, shape=(1800, 3600)) -> np.ndarray:
    """Config 2 (ATM-like): GRF(beta~U(1.5,3.5)) x 10^U(-3,3) + U(-1e3,1e3);
    every 10th field piecewise-constant with sharp fronts (6 quantile levels of a GRF(3))."""
    rng = np.random.default_rng([2, i, 0])
    beta = rng.uniform(1.5, 3.5)
    scale = 10.0 ** rng.uniform(-3.0, 3.0)
    offset = rng.uniform(-1e3, 1e3)
    if i % 10 == 0:
        g = grf(shape, 3.0, rng)
        edges = np.quantile(g, [1 / 6, 2 / 6, 3 / 6, 4 / 6, 5 / 6])
        lev = np.searchsorted(edges, g)
        vals = rng.uniform(-1.0, 1.0, size=6)
        g = vals[lev]
    else:
        g = grf(shape, beta, rng)
    return (g * scale + offset).astype(np.float32)


# --------------------------------------------------------------------------- C3
def c3_field(i: int, shape=(100, 500, 500)) -> np.ndarray:
    """Config 3 (Hurricane-like): tanh vortex + a*V0*GRF(3) turbulence + 1e-4-relative noise;
    fields 5-6 are zero-heavy (exactly 0 on a coherent 30%)."""
    rng = np.random.default_rng([3, i, 0])
    nz, ny, nx = shape
    cy = ny / 2 + rng.uniform(-0.05, 0.05) * ny
    cx = nx / 2 + rng.uniform(-0.05, 0.05) * nx
    r0 = rng.uniform(20.0, 60.0) * min(ny, nx) / 500.0
    H = rng.uniform(30.0, 100.0) * nz / 100.0
    V0 = rng.uniform(20.0, 60.0)
    z = np.arange(nz, dtype=np.float64).reshape(nz, 1, 1)
    yy = (np.arange(ny, dtype=np.float64) - cy).reshape(1, ny, 1)
    xx = (np.arange(nx, dtype=np.float64) - cx).reshape(1, 1, nx)
    r = np.sqrt(yy ** 2 + xx ** 2)
    prof = np.tanh(r / r0) * np.exp(-z / H)          # (nz, ny, nx)
    sin_t = np.where(r > 0, yy / np.where(r > 0, r, 1.0), 0.0)
    cos_t = np.where(r > 0, xx / np.where(r > 0, r, 1.0), 0.0)
    amps = {0: 0.1, 1: 0.1, 7: 0.05, 8: 0.1, 9: 0.2, 10: 0.3, 11: 0.4, 12: 0.5}
    if i in (0, 7, 8, 9, 10, 11, 12):
        f = -V0 * prof * sin_t + amps[i] * V0 * grf(shape, 3.0, rng)
    elif i == 1:
        f = V0 * prof * cos_t + amps[i] * V0 * grf(shape, 3.0, rng)
    elif i == 2:
        f = 0.1 * V0 * grf(shape, 3.0, rng)
    elif i == 3:
        f = 1000.0 - 50.0 * prof + 0.0 * z
    elif i == 4:
        f = 300.0 - 0.5 * z * (100.0 / nz) + 0.2 * V0 * prof * cos_t
    else:  # 5, 6: zero-heavy (QICE / PRECIP-like)
        s = prof * (1.0 + 0.3 * grf(shape, 3.0, rng))
        f = np.maximum(0.0, s - np.quantile(s, 0.30))
    f = np.broadcast_to(f, shape).astype(np.float64)
    if i not in (5, 6):
        vr = f.max() - f.min()
        f = f + rng.normal(0.0, 1e-4 * vr if vr > 0 else 1e-4, size=shape)
    return np.ascontiguousarray(f, dtype=np.float32)


# --------------------------------------------------------------------------- C4
def c4_field(i: int, shape=(512, 512, 512)) -> np.ndarray:
    """Config 4 (NYX-like): f0 lognormal exp(sG*GRF(2.5)) with VR ~ 1e6 and median ~ 1;
    f1-f3 = 300*GRF(3) velocities; f4-f5 = 1e4*exp(0.5*GRF(3.5)) temperatures."""
    rng = np.random.default_rng([4, i, 0])
    if i == 0:
        g = grf(shape, 2.5, rng)
        s = np.log(1e6) / g.max()
        f = np.exp(s * g)
    elif i in (1, 2, 3):
        f = 300.0 * grf(shape, 3.0, rng)
    else:
        f = 1e4 * np.exp(0.5 * grf(shape, 3.5, rng))
    return f.astype(np.float32)


# --------------------------------------------------------------------------- C5
def c5_field(mix_idx: int, shape=(1024, 1024, 1024)) -> np.ndarray:
    """Config 5 (stress): w*N(0,1) + (1-w)*ramp, w = (0, 0.5, 1)[mix_idx],
    ramp = 8(i+j+k)/(3(n-1)) - 4; drawn per 4-plane slab with its own seed."""
    w = (0.0, 0.5, 1.0)[mix_idx]
    n0, n1, n2 = shape
    out = np.empty(shape, np.float32)
    den = 3.0 * max(max(shape) - 1, 1)
    jk = (np.arange(n1, dtype=np.float64).reshape(n1, 1) + np.arange(n2, dtype=np.float64))
    for sl in range(0, n0, 4):
        rng = np.random.default_rng([5, mix_idx, sl // 4])
        m = min(4, n0 - sl)
        i = np.arange(sl, sl + m, dtype=np.float64).reshape(m, 1, 1)
        ramp = 8.0 * (i + jk) / den - 4.0
        z = rng.standard_normal((m, n1, n2)) if w > 0 else 0.0
        out[sl:sl + m] = (w * z + (1.0 - w) * ramp).astype(np.float32)
    return out


def make_field(config: int, i: int, shape=None) -> np.ndarray:
    gen = {1: lambda i, s: c1_field(s or (256, 256), seed=i),
           2: lambda i, s: c2_field(i, s or CONFIGS[2]["shape"]),
           3: lambda i, s: c3_field(i, s or CONFIGS[3]["shape"]),
           4: lambda i, s: c4_field(i, s or CONFIGS[4]["shape"]),
           5: lambda i, s: c5_field(i, s or CONFIGS[5]["shape"])}[config]
    return gen(i, shape)


def config_fields(config: int, shape=None, n_fields=None):
    n = CONFIGS[config]["n_fields"] if n_fields is None else n_fields
    for i in range(n):
        yield make_field(config, i, shape)
