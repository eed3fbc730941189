"""Seeded synthetic inputs for the PGET hot path (configs 1-5 of BASELINE.json).

This module is shared by the oracle tests, the GPU parity tests and bench.py.
It holds NONE of the method's arithmetic (no ray tracing, no attenuation, no
derivatives): only phantom rasterisation, random directions/weights and the
Poisson corruption of a sinogram that the caller computed elsewhere.

Recipes follow SURVEY.md §8(d) (phantom table, seeds, draw order) and the
readings Q14, Q15, Q20 of SURVEY.md §8(c.3); the shapes borrow the paper's
9x9 lattice (§3.3 "Training setup"), a hexagonal VVER-440-like
assembly (§4.2) and 2x91 detectors (§2).
Draw order per seed: rod lambda values (lattice order), then rod mu values
(cfg 4 only), then the special-rod choice, then directions, then noise.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

__all__ = [
    "CONFIGS", "Config", "geometry_desc", "make_phantom", "make_phantom_prime",
    "rod_directions", "white_directions", "white_weights", "initial_guess",
    "poisson_noise", "rng_for", "disk_phantom", "prior_masks",
]


@dataclass(frozen=True)
class Config:
    cid: int
    n_px: int
    n_angles: int
    n_subrays: int
    batch: int
    lattice: str          # "sq9", "sq17", "hex127"
    seed: int
    noise_peak: float | None  # Poisson peak counts (None = no noise)
    lm: bool               # the config runs an LM iteration
    n_det: int = 91
    n_banks: int = 2
    subray_sigma: float = 0.4
    step_px: float = 0.5
    bank1_shift: float = 0.0
    alpha: float = 1e-3
    n_cg: int = 20


CONFIGS = {
    1: Config(1, 64, 90, 1, 1, "sq9", 1, None, False),
    2: Config(2, 128, 360, 5, 1, "sq9", 2, 1e4, True),
    3: Config(3, 256, 360, 9, 1, "sq17", 3, 1e4, True),
    4: Config(4, 256, 720, 9, 1, "hex127", 4, 1e4, True),
    5: Config(5, 128, 360, 5, 64, "sq9", 5000, None, False),
}


def geometry_desc(cfg: Config | int, **over) -> dict:
    """Geometry descriptor (the fields of pget_geometry_desc)."""
    if isinstance(cfg, int):
        cfg = CONFIGS[cfg]
    d = dict(n_px=cfg.n_px, n_angles=cfg.n_angles, n_banks=cfg.n_banks, n_det=cfg.n_det,
             n_subrays=cfg.n_subrays, subray_sigma=cfg.subray_sigma, step_px=cfg.step_px,
             bank1_shift=cfg.bank1_shift, batch=cfg.batch)
    d.update(over)
    return d


def rng_for(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


# ----------------------------------------------------------------------------- lattices
def _lattice(kind: str):
    """Rod centres (x, y) in lattice order and the rod radius."""
    if kind == "sq9":
        c = [((ix - 4) * 0.2, (iy - 4) * 0.2) for iy in range(9) for ix in range(9)]
        return np.array(c), 0.08, None
    if kind == "sq17":
        c = [((ix - 8) * 0.11, (iy - 8) * 0.11) for iy in range(17) for ix in range(17)]
        guide = set()
        for a in (0, 3, 6):
            for b in (0, 3, 6):
                if a == 0 and b == 0:
                    guide.add((0, 0))
                    continue
                for sa in ((1, -1) if a else (1,)):
                    for sb in ((1, -1) if b else (1,)):
                        guide.add((sa * a, sb * b))
        gidx = sorted((gy + 8) * 17 + (gx + 8) for (gx, gy) in guide)
        assert len(gidx) == 25
        return np.array(c), 0.045, gidx
    if kind == "hex127":
        c = []
        s3 = math.sqrt(3.0) / 2.0
        for b in range(-6, 7):
            for a in range(-6, 7):
                if max(abs(a), abs(b), abs(a + b)) <= 6:
                    c.append((a * 0.15 + b * 0.075, b * 0.15 * s3))
        assert len(c) == 127
        return np.array(c), 0.06, None
    raise ValueError(kind)


def _area_fractions(n_px: int, centres: np.ndarray, radius: float, ss: int = 8):
    """Per rod: (rows, cols, fraction) of the pixels it covers, by ss x ss supersampling
    of each pixel (reading Q15: "generated at twice the spatial resolution",
    PAPER.md:326).  Pixel (iy, ix) is centred at (-1+(ix+1/2)h, -1+(iy+1/2)h)."""
    h = 2.0 / n_px
    off = (np.arange(ss) + 0.5) / ss
    out = []
    r2 = radius * radius
    for (cx, cy) in centres:
        ix0 = max(0, int(math.floor((cx - radius + 1.0) / h)) - 1)
        ix1 = min(n_px - 1, int(math.floor((cx + radius + 1.0) / h)) + 1)
        iy0 = max(0, int(math.floor((cy - radius + 1.0) / h)) - 1)
        iy1 = min(n_px - 1, int(math.floor((cy + radius + 1.0) / h)) + 1)
        if ix1 < ix0 or iy1 < iy0:
            out.append((np.zeros(0, int), np.zeros(0, int), np.zeros(0)))
            continue
        ixs = np.arange(ix0, ix1 + 1)
        iys = np.arange(iy0, iy1 + 1)
        xs = -1.0 + (ixs[:, None] + off[None, :]) * h          # [nx, ss]
        ys = -1.0 + (iys[:, None] + off[None, :]) * h          # [ny, ss]
        dx2 = (xs - cx) ** 2
        dy2 = (ys - cy) ** 2
        inside = (dy2[:, None, :, None] + dx2[None, :, None, :]) <= r2   # [ny, nx, ss, ss]
        frac = inside.mean(axis=(2, 3))
        yy, xx = np.nonzero(frac > 0)
        out.append((iys[yy], ixs[xx], frac[yy, xx]))
    return out


def _raster(n_px, fracs, rod_vals, bg):
    img = np.full((n_px, n_px), bg, dtype=np.float64)
    for (rows, cols, f), v in zip(fracs, rod_vals):
        img[rows, cols] = bg + f * (v - bg)
    return img


def _rod_values(cfg: Config, rng: np.random.Generator):
    """Rod (lambda, mu) values and the special-rod indices, in the fixed draw order."""
    centres, radius, guide = _lattice(cfg.lattice)
    n = len(centres)
    lam = rng.uniform(0.5, 1.5, size=n)
    if cfg.lattice == "hex127":
        mu = rng.uniform(0.4, 0.6, size=n)
        special = rng.choice(n, 7, replace=False)
        lam[special] = 0.0
        mu[special] = 0.3
    elif cfg.lattice == "sq17":
        mu = np.full(n, 0.5)
        lam[guide] = 0.0
        mu[guide] = 0.05
        eligible = np.array([i for i in range(n) if i not in set(guide)])
        special = eligible[rng.choice(len(eligible), 5, replace=False)]
        lam[special] = 0.0
        mu[special] = 0.05
    else:
        mu = np.full(n, 0.5)
        special = rng.choice(n, 3, replace=False)
        lam[special] = 0.0
    return centres, radius, lam, mu


def _member_seed(cfg: Config, b: int) -> int:
    return cfg.seed + b if cfg.batch > 1 else cfg.seed


def make_phantom(cfg: Config | int, n_px: int | None = None):
    """Phantom (lam, mu) as float32 arrays [B][N][N] (row = y, col = x)."""
    if isinstance(cfg, int):
        cfg = CONFIGS[cfg]
    n = n_px or cfg.n_px
    lams, mus = [], []
    for b in range(cfg.batch):
        rng = rng_for(_member_seed(cfg, b))
        centres, radius, lv, mv = _rod_values(cfg, rng)
        fr = _area_fractions(n, centres, radius)
        lams.append(_raster(n, fr, lv, 0.0))
        mus.append(_raster(n, fr, mv, 0.05))
    return np.stack(lams).astype(np.float32), np.stack(mus).astype(np.float32)


def make_phantom_prime(cfg: Config | int, n_px: int | None = None):
    """u' of SURVEY §8(d): the same lattice and special rods, rod values redrawn
    (seed + 100000).  Used for residual-like VJP weights w = F(u') - F(u)."""
    if isinstance(cfg, int):
        cfg = CONFIGS[cfg]
    n = n_px or cfg.n_px
    lams, mus = [], []
    for b in range(cfg.batch):
        rng = rng_for(_member_seed(cfg, b))
        centres, radius, lv, mv = _rod_values(cfg, rng)
        rng2 = rng_for(_member_seed(cfg, b) + 100000)
        lv2 = np.where(lv > 0, rng2.uniform(0.5, 1.5, size=len(lv)), 0.0)
        mv2 = np.where(mv >= 0.4, mv * rng2.uniform(0.95, 1.05, size=len(mv)), mv)
        fr = _area_fractions(n, centres, radius)
        lams.append(_raster(n, fr, lv2, 0.0))
        mus.append(_raster(n, fr, mv2, 0.05))
    return np.stack(lams).astype(np.float32), np.stack(mus).astype(np.float32)


def rod_directions(cfg: Config | int, n_px: int | None = None, seed_offset: int = 7):
    """Rod-structured directions (the shape of LM steps, reading Q17):
    per-rod U[-0.5,0.5] (lambda) and U[-0.05,0.05] (mu) times the rod's area fraction."""
    if isinstance(cfg, int):
        cfg = CONFIGS[cfg]
    n = n_px or cfg.n_px
    dl, dm = [], []
    for b in range(cfg.batch):
        centres, radius, _ = _lattice(cfg.lattice)
        rng = rng_for(_member_seed(cfg, b) * 1000 + seed_offset)
        a = rng.uniform(-0.5, 0.5, size=len(centres))
        m = rng.uniform(-0.05, 0.05, size=len(centres))
        fr = _area_fractions(n, centres, radius)
        dl.append(_raster(n, fr, a, 0.0))
        dm.append(_raster(n, fr, m, 0.0))
    return np.stack(dl).astype(np.float32), np.stack(dm).astype(np.float32)


def white_directions(shape, seed: int):
    """White-noise directions: dlam ~ U[-1,1], dmu ~ U[-0.1,0.1] (rel-L2/adjoint only)."""
    rng = rng_for(seed)
    return (rng.uniform(-1, 1, size=shape).astype(np.float32),
            rng.uniform(-0.1, 0.1, size=shape).astype(np.float32))


def white_weights(shape, seed: int):
    """w ~ N(0,1) sinogram-shaped weights (rel-L2/adjoint only)."""
    return rng_for(seed).standard_normal(size=shape).astype(np.float32)


def prior_masks(cfg: Config | int, n_px: int | None = None, margin_px: float = 1.0):
    """Geometry-prior masks (P1 = diag(m_lam), P2 = diag(m_mu), reading R-prior):
    1 on pixels whose centre lies farther than the rod radius + margin_px pixels from every lattice
    position of the configuration (rod or not: no position is assumed filled a priori), else 0.
    float32 [B][N][N], the same for both parts and every member."""
    if isinstance(cfg, int):
        cfg = CONFIGS[cfg]
    n = n_px or cfg.n_px
    centres, radius, _ = _lattice(cfg.lattice)
    h = 2.0 / n
    c = -1.0 + (np.arange(n) + 0.5) * h
    near = np.zeros((n, n), dtype=bool)
    r = radius + margin_px * h
    for (cx, cy) in centres:
        near |= (c[None, :] - cx) ** 2 + (c[:, None] - cy) ** 2 <= r * r
    m = np.where(near, 0.0, 1.0).astype(np.float32)
    m = np.broadcast_to(m, (cfg.batch, n, n)).copy()
    return m, m.copy()


def initial_guess(n_px: int, batch: int = 1):
    """Reading Q20: u0 = (0.75, 0.30) on pixels whose centre lies in the unit disk."""
    h = 2.0 / n_px
    c = -1.0 + (np.arange(n_px) + 0.5) * h
    disk = (c[None, :] ** 2 + c[:, None] ** 2) <= 1.0
    lam = np.where(disk, 0.75, 0.0).astype(np.float32)
    mu = np.where(disk, 0.30, 0.0).astype(np.float32)
    return (np.broadcast_to(lam, (batch, n_px, n_px)).copy(),
            np.broadcast_to(mu, (batch, n_px, n_px)).copy())


def poisson_noise(y_clean: np.ndarray, peak: float, seed: int):
    """Reading Q14: y = Poisson(c * y_clean) / c with c = peak / max(y_clean).
    y_clean is computed by the caller (the oracle in tests, the library in bench)."""
    y = np.asarray(y_clean, dtype=np.float64)
    c = peak / max(float(y.max()), 1e-30)
    rng = rng_for(seed + 555)
    return (rng.poisson(np.clip(y, 0, None) * c) / c).astype(np.float32)


def disk_phantom(n_px: int, radius: float = 0.5, lam0: float = 1.0, mu0: float = 0.5,
                 centre=(0.0, 0.0)):
    """Pixelised uniform disk (area fractions by 8x8 supersampling), float64 [1][N][N].
    Used by the closed-form pins P2/P4 (north star: g(s) = lam0 (1 - e^{-mu0 2 sqrt(R^2-s^2)})/mu0)."""
    fr = _area_fractions(n_px, np.array([centre]), radius)
    lam = _raster(n_px, fr, [lam0], 0.0)
    mu = _raster(n_px, fr, [mu0], 0.0)
    return lam[None], mu[None]
