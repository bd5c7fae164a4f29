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


NEAR = 1e-5
PARITY: dict = {}  # observed mismatch counts by test (written to profiles/parity_r02.json, conftest.py)


def record(name: str, counts: dict) -> dict:
    PARITY[name] = counts
    return counts


def mismatch_classes(mism: np.ndarray, pre: np.ndarray, slm, pred: np.ndarray | None = None,
                     rounding: float = 2e-7) -> dict:
    """Classify level mismatches against the oracle's pre-quantisation field
    `pre` (the north-star exception and the low-|f| class, see
    tests/test_gpu_lockstep.py):
      near       the oracle's angle is within 1e-5 rad of a threshold;
      lowf       within 1e-5 rad + 6 x the transform's rounding (rounding x RMS |f|) / |f|;
      propagated (with `pred`, the GPU's own pre-quantisation field predicted
                 from its previous iteration) the prediction is near a
                 threshold by the same rule or quantises differently.
    Returns counts; "bad" must be 0."""
    d = phase_threshold_distance(pre, slm)
    mag = np.abs(pre)
    floor = rounding * float(np.sqrt(np.mean(mag ** 2)))
    near = d < NEAR
    lowf = ~near & (d < NEAR + 6.0 * floor / np.maximum(mag, 1e-300))
    out = {"mismatch": int(mism.sum()), "near": int((mism & near).sum()), "lowf": int((mism & lowf).sum())}
    ok = near | lowf
    if pred is not None:
        dp = phase_threshold_distance(pred, slm)
        mp = np.abs(pred)
        prop = ~ok & ((dp < NEAR + 6.0 * floor / np.maximum(mp, 1e-300)) |
                      (quantise_phase_levels(pred, slm) != quantise_phase_levels(pre, slm)))
        out["propagated"] = int((mism & prop).sum())
        ok = ok | prop
    out["bad"] = int((mism & ~ok).sum())
    return out


def quantise_phase_levels(f: np.ndarray, slm) -> np.ndarray:
    """Phase-mode quantiser decision (quantise.hpp:175-198) in double."""
    d = np.arctan2(f.imag, f.real) - slm.min_arg
    d = d - TWO_PI * np.floor(d / TWO_PI)
    L = slm.levels
    if slm.full_circle:
        k = np.floor(d * (L / TWO_PI) + 0.5).astype(np.int64)
        return np.where(k >= L, 0, k)
    rng = slm.max_arg - slm.min_arg
    spac = rng / (L - 1)
    k = np.minimum(np.floor(d / spac + 0.5).astype(np.int64), L - 1)
    return np.where(d <= rng, k, np.where(d - rng <= TWO_PI - d, L - 1, 0))
