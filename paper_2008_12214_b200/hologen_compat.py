"""Drop-in for the reference's Python module ``hologen`` (proj/python:
bindings.cpp:150-260, hologen/__init__.py) on the GPU hot path.

Same function names, arguments, defaults and return dictionaries as the
pybind11 module for the functions on the IFTA / OSPR path:
``fft_forward``, ``fft_inverse``, ``quantise``, ``gs``, ``wgs``, ``lt``,
``ospr``, ``adaptive_ospr``, ``mse``.  Arrays are numpy (height, width),
complex128 fields and float64 images like the reference's, computed in
double on the B200 as the reference module computes them: the transforms by
hgc_fft2d_f64 and the algorithms by the device f64 loops (hgc_ifta_run_f64 /
hgc_ospr_run_f64, the reference's double arithmetic per pixel).  The
float32 hot path is ``paper_2008_12214_b200.run_*``.
Holographic search and SSIM (``direct_search``, ``simulated_annealing``,
``ssim``) are not on the hot path and are not provided.

    import paper_2008_12214_b200.hologen_compat as hologen
    run = hologen.gs(target, iterations=25, levels=256, seed=1)
"""
from __future__ import annotations

import numpy as np

from . import api
from .types import IftaConfig, IftaVariant, MetricConfig, OsprConfig, OsprVariant, SlmSpec, TargetSpec

__version__ = "0.1.0"

__all__ = ["__version__", "adaptive_ospr", "fft_forward", "fft_inverse", "gs", "lt", "mse", "ospr", "quantise",
           "wgs"]


def _field(a) -> np.ndarray:
    a = np.asarray(a)
    if a.ndim != 2:
        raise ValueError("expected a 2-D complex array")  # bindings.cpp:20
    return a


def _image(a) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    if a.ndim != 2:
        raise ValueError("expected a 2-D real array")  # bindings.cpp:29
    return a


def _slm(levels: int) -> SlmSpec:  # bindings.cpp slm_from_levels
    return SlmSpec.binary_phase() if levels == 2 else SlmSpec.full_circle_phase(levels)


def _target(amplitude, phase_freedom: bool) -> TargetSpec:  # bindings.cpp target_from
    t = TargetSpec(_image(amplitude))
    t.freedoms.phase = bool(phase_freedom)
    return t


def _report(rep) -> dict:  # bindings.cpp report_dict
    return {"algorithm": rep.algorithm, "hologram": np.asarray(rep.hologram, np.complex128),
            "replay": np.asarray(rep.replay, np.complex128), "final_error": float(rep.final_error),
            "evaluations": int(rep.evaluations),
            "trace": [(int(i), float(v)) for i, v in rep.trace.points]}


def fft_forward(field) -> np.ndarray:
    """Unitary forward transform (aperture plane to replay field), in double on the GPU."""
    return api.fft_forward(np.asarray(_field(field), np.complex128))


def fft_inverse(field) -> np.ndarray:
    """Unitary inverse transform (replay field to aperture plane), in double on the GPU."""
    return api.fft_inverse(np.asarray(_field(field), np.complex128))


def quantise(field, levels: int = 256) -> np.ndarray:
    """Project every pixel onto the nearest allowed modulator state (levels == 2
    means binary phase {0, pi}, otherwise a full phase circle).  Decisions in
    double; the states are the float32 hot-path table widened to double."""
    return api.quantise_field(_field(field), _slm(levels)).astype(np.complex128)


def _ifta(variant, target, iterations, levels, seed, phase_freedom, clamp_lo=0.1, clamp_hi=10.0, lt_fraction=0.1):
    cfg = IftaConfig(variant=variant, iterations=iterations, slm=_slm(levels), target=_target(target, phase_freedom),
                     seed=seed, weight_clamp_lo=clamp_lo, weight_clamp_hi=clamp_hi, lt_initial_fraction=lt_fraction)
    return _report(api.run_ifta_f64(cfg))


def gs(target, iterations: int = 25, levels: int = 256, seed: int = 0, phase_freedom: bool = True) -> dict:
    """Iterative transform algorithm with hard replay amplitude substitution."""
    return _ifta(IftaVariant.GS, target, iterations, levels, seed, phase_freedom)


def wgs(target, iterations: int = 25, levels: int = 256, seed: int = 0, phase_freedom: bool = True,
        clamp_lo: float = 0.1, clamp_hi: float = 10.0) -> dict:
    """Weighted iterative transform algorithm with clamped per-pixel gains."""
    return _ifta(IftaVariant.WeightedGS, target, iterations, levels, seed, phase_freedom, clamp_lo, clamp_hi)


def lt(target, iterations: int = 25, levels: int = 256, seed: int = 0, phase_freedom: bool = True,
       initial_fraction: float = 0.1) -> dict:
    """Iterative transform algorithm with a growing active target region."""
    return _ifta(IftaVariant.LiuTaghizadeh, target, iterations, levels, seed, phase_freedom,
                 lt_fraction=initial_fraction)


def _ospr(variant, target, subframes, levels, seed, phase_freedom, gain) -> dict:  # bindings.cpp run_ospr_py
    cfg = OsprConfig(variant=variant, subframes=subframes, slm=_slm(levels), target=_target(target, phase_freedom),
                     seed=seed, feedback_gain=gain)
    run = api.run_ospr_f64(cfg)
    d = _report(run.report)
    d["frames"] = [np.asarray(f, np.complex128) for f in run.set.frames]
    d["mean_intensity"] = np.asarray(run.set.mean_intensity, np.float64)
    d["per_frame_mse"] = [float(v) for v in run.set.per_frame_mse]
    return d


def ospr(target, subframes: int = 24, levels: int = 2, seed: int = 0, phase_freedom: bool = True) -> dict:
    """One-step phase retrieval: independent random-phase subframes, time averaged."""
    return _ospr(OsprVariant.Ospr, target, subframes, levels, seed, phase_freedom, 1.0)


def adaptive_ospr(target, subframes: int = 24, levels: int = 2, seed: int = 0, phase_freedom: bool = True,
                  gain: float = 1.0) -> dict:
    """OSPR with per-subframe feedback on the running intensity."""
    return _ospr(OsprVariant.AdaptiveOspr, target, subframes, levels, seed, phase_freedom, gain)


def mse(target, replay, mask=None, phase_sensitive: bool = False, scale_free: bool = False) -> float:
    """Mean squared error between the target amplitude and |replay|."""
    m = None if mask is None else (np.asarray(mask) != 0)
    return api.mse(_image(target), np.asarray(replay).astype(np.complex64),
                   MetricConfig(phase_sensitive=phase_sensitive, scale_free=scale_free, mask=m))
