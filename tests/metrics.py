"""Parity metrics of SURVEY.md §8(c) Q17 (shared by the oracle and GPU tests)."""
import numpy as np


def rel_l2(x, o):
    x = np.asarray(x, np.float64).ravel()
    o = np.asarray(o, np.float64).ravel()
    d = np.linalg.norm(o)
    return float(np.linalg.norm(x - o) / (d if d > 0 else 1.0))


def max_rel(x, o, floor=1e-3):
    """max_i |x_i - o_i| / max(|o_i|, floor * ||o||_inf)."""
    x = np.asarray(x, np.float64).ravel()
    o = np.asarray(o, np.float64).ravel()
    m = np.abs(o).max() if o.size else 0.0
    den = np.maximum(np.abs(o), floor * m)
    den = np.where(den > 0, den, 1.0)
    return float((np.abs(x - o) / den).max()) if o.size else 0.0
