"""Shared helpers for the parity tests (oracle comparison rules)."""
from __future__ import annotations

import numpy as np

TWO_PI = 6.283185307179586476925286766559


def phase_threshold_distance(field: np.ndarray, slm) -> np.ndarray:
    """Distance (rad) of each pixel's pre-quantisation angle to the nearest
    decision boundary of a phase-mode SLM (quantise.hpp:175-198), computed in
    double from the complex64 values."""
    ang = np.arctan2(field.imag.astype(np.float64), field.real.astype(np.float64))
    d = ang - slm.min_arg
    d = d - TWO_PI * np.floor(d / TWO_PI)
    spac = TWO_PI / slm.levels if slm.full_circle else (slm.max_arg - slm.min_arg) / (slm.levels - 1)
    u = d / spac
    dist = np.abs((u - np.floor(u)) - 0.5) * spac
    if not slm.full_circle:
        rng = slm.max_arg - slm.min_arg
        dist = np.minimum(dist, np.abs(d - (np.pi + rng / 2)))
        dist = np.minimum(dist, np.minimum(d, TWO_PI - d))
    return dist


def level_mismatches(got: np.ndarray, ref: np.ndarray) -> np.ndarray:
    return np.asarray(got).astype(np.int64) != np.asarray(ref).astype(np.int64)


def rel(a: float, b: float) -> float:
    return abs(a - b) / max(abs(b), 1e-300)
