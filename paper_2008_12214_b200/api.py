"""Reference-shaped entry points over the B200 C ABI.

Mirrors proj/include/hologen (run_gs / run_weighted_gs / run_liu_taghizadeh /
run_ifta, run_ospr / run_adaptive_ospr / run_ospr_variant, fft_forward /
fft_inverse, Quantiser / quantise_field, seed_random_phase, mse,
make_fresnel_phase / Propagator, subframe_mse_statistic) with the same
argument meaning and error behaviour (ValueError for std::invalid_argument).
All arithmetic runs in the sm_100a kernels; nothing here computes on the CPU
beyond marshalling.  Batched forms (``run_ifta_batch``, ``run_ospr_batch``)
and device-resident plans (``IftaPlan``, ``OsprPlan``) are the B200-native
extensions used for throughput (the reference's cmd_batch job pool,
runner.cpp:365-421).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check, lib
from .types import (FresnelParams, IftaConfig, IftaVariant, InitPhase, MetricConfig, MetricTrace, OsprConfig,
                    OsprRun, OsprVariant, PhaseProfile, RunReport, SlmMode, SlmSpec, SubframeSet)


def _p(a):
    return None if a is None else a.ctypes.data


def _slm(spec: SlmSpec, keep: list) -> _lib.HgcSlm:
    s = _lib.HgcSlm()
    s.mode = int(spec.mode)
    s.levels = int(spec.levels)
    s.min_arg = float(spec.min_arg)
    s.max_arg = float(spec.max_arg)
    s.full_circle = int(bool(spec.full_circle))
    s.min_amp = float(spec.min_amp)
    s.max_amp = float(spec.max_amp)
    if spec.illumination is not None:
        il = np.ascontiguousarray(spec.illumination, dtype=np.complex128)
        keep.append(il)
        s.illumination = il.ctypes.data
    return s


def _fresnel(p: FresnelParams | None):
    if p is None:
        return None
    f = _lib.HgcFresnel(p.wavelength, p.distance, p.pixel_pitch_x, p.pixel_pitch_y)
    return C.byref(f)


# ------------------------------------------------------------- Propagator
class Propagator:
    """Propagator<float> (propagation.hpp:60-116): Fourier, or Fresnel with
    the quadratic phase Q applied around the transform."""

    def __init__(self, fresnel: FresnelParams | None = None, nx: int = 0, ny: int = 0):
        self.params = fresnel
        self.nx, self.ny = nx, ny

    @staticmethod
    def fourier() -> "Propagator":
        return Propagator()

    @staticmethod
    def fresnel(nx: int, ny: int, params: FresnelParams) -> "Propagator":
        params.validate()
        return Propagator(params, nx, ny)

    def is_fresnel(self) -> bool:
        return self.params is not None

    def _check(self, f):
        if self.params is not None and (f.shape[1] != self.nx or f.shape[0] != self.ny):
            raise ValueError("Propagator: field size does not match Fresnel phase")

    def forward(self, f: np.ndarray) -> np.ndarray:
        self._check(f)
        return _fft2d(f, -1, self.params)

    def inverse(self, F: np.ndarray) -> np.ndarray:
        self._check(F)
        return _fft2d(F, +1, self.params)

    def aperture_factor(self, x: int, y: int) -> complex:
        if self.params is None:
            return 1 + 0j
        return complex(make_fresnel_phase(self.nx, self.ny, self.params)[y, x])


def _fft2d(f: np.ndarray, sign: int, fresnel: FresnelParams | None = None) -> np.ndarray:
    if fresnel is None and np.asarray(f).dtype == np.complex128:  # fft_forward<double>
        a = np.ascontiguousarray(f)
        a3 = a[None] if a.ndim == 2 else a
        b, ny, nx = a3.shape
        out = np.empty_like(a3)
        check(lib.hgc_fft2d_f64(nx, ny, sign, b, _p(a3), _p(out)))
        return out[0] if a.ndim == 2 else out
    a = np.ascontiguousarray(f, dtype=np.complex64)
    if a.ndim == 2:
        a = a[None]
    b, ny, nx = a.shape
    out = np.empty_like(a)
    if fresnel is None:
        check(lib.hgc_fft2d(nx, ny, sign, b, _p(a), _p(out)))
    else:
        check(lib.hgc_propagate(nx, ny, sign, _fresnel(fresnel), b, _p(a), _p(out)))
    return out.reshape(f.shape)


def fft_forward(f: np.ndarray) -> np.ndarray:
    """fft_forward<T> (fft.hpp:93-102): unitary, -i exponent; T = float for
    complex64 input (the hot-path transform), double for complex128."""
    return _fft2d(f, -1)


def fft_inverse(F: np.ndarray) -> np.ndarray:
    """fft_inverse<T> (fft.hpp:104-113): unitary, +i exponent; complex64 -> float, complex128 -> double."""
    return _fft2d(F, +1)


def make_fresnel_phase(nx: int, ny: int, p: FresnelParams) -> np.ndarray:  # propagation.hpp:36-54
    q = np.empty((ny, nx), np.complex64)
    f = _lib.HgcFresnel(p.wavelength, p.distance, p.pixel_pitch_x, p.pixel_pitch_y)
    check(lib.hgc_fresnel_phase(nx, ny, C.byref(f), _p(q)))
    return q


def fresnel_forward(f: np.ndarray, p: FresnelParams) -> np.ndarray:  # propagation.hpp:119-125
    return Propagator.fresnel(f.shape[-1], f.shape[-2], p).forward(f)


def fresnel_inverse(F: np.ndarray, p: FresnelParams) -> np.ndarray:  # propagation.hpp:127-133
    return Propagator.fresnel(F.shape[-1], F.shape[-2], p).inverse(F)


# -------------------------------------------------------------- quantiser
class Quantiser:
    """Quantiser<float> (quantise.hpp:136-231)."""

    def __init__(self, spec: SlmSpec, nx: int, ny: int):
        spec.validate()
        if spec.illumination is not None and np.asarray(spec.illumination).shape != (ny, nx):
            raise ValueError("Quantiser: illumination dimensions mismatch")
        self.spec, self.nx, self.ny = spec, nx, ny
        canon = allowed_states_f32(spec)
        self.states = canon
        il = None if spec.illumination is None else np.asarray(spec.illumination, np.complex128)
        self._illum = None if il is None else il.astype(np.complex64)
        self._illum_unit = None if il is None else (il / np.abs(il)).astype(np.complex64)

    def level_count(self) -> int:
        return int(self.spec.levels)

    def apply(self, f: np.ndarray, levels_out: bool = False):
        """Snap in place; returns level indices when levels_out."""
        if f.shape[-2:] != (self.ny, self.nx):
            raise ValueError("Quantiser: field dimensions mismatch")
        a = np.ascontiguousarray(f, dtype=np.complex64)
        batch = a.size // (self.nx * self.ny)
        lv = np.empty(a.shape, np.int32) if levels_out else None
        keep = []
        check(lib.hgc_quantise(C.byref(_slm(self.spec, keep)), self.nx, self.ny, batch, _p(a), _p(lv)))
        if a is not f:
            f[...] = a
        return lv

    def decide(self, f: np.ndarray) -> np.ndarray:
        """Level index of every pixel of a field (Quantiser::decide)."""
        g = np.array(f, dtype=np.complex64, copy=True)
        return self.apply(g, levels_out=True)

    def state_value(self, i: int, k: int) -> complex:
        s = self.states[k]
        if self.spec.mode == SlmMode.Phase:
            return s if self._illum is None else _cmul_f32(self._illum.ravel()[i], s)
        return s if self._illum_unit is None else _cmul_f32(self._illum_unit.ravel()[i], s)


def _cmul_f32(a, b) -> np.complex64:
    ar, ai, br, bi = (np.float32(a.real), np.float32(a.imag), np.float32(b.real), np.float32(b.imag))
    return np.complex64(complex(ar * br - ai * bi, ar * bi + ai * br))


def allowed_states_f32(spec: SlmSpec) -> np.ndarray:
    """(T)allowed_states(spec) as the quantiser stores them (quantise.hpp:147-149)."""
    import math
    spac = spec.spacing()
    out = np.empty(spec.levels, np.complex64)
    for k in range(spec.levels):
        if spec.mode == SlmMode.Phase:
            a = spec.min_arg + k * spac
            out[k] = complex(np.float32(math.cos(a)), np.float32(math.sin(a)))
        else:
            out[k] = complex(np.float32(spec.min_amp + k * spac), 0.0)
    return out


def quantise_field(field: np.ndarray, spec: SlmSpec) -> np.ndarray:  # quantise.hpp:234-243
    if not np.all(np.isfinite(field)):
        raise ValueError("quantise_field: field contains non-finite values")
    out = np.array(field, dtype=np.complex64, copy=True)
    Quantiser(spec, field.shape[-1], field.shape[-2]).apply(out)
    return out


# -------------------------------------------------------------------- rng
def fork_seed(seed: int, stream: int = 0) -> int:
    """Engine seed of Rng(seed).fork(stream) (rng.hpp:42-44)."""
    return int(lib.hgc_fork_seed(seed, stream))


def seed_random_phase(amp: np.ndarray, seed: int, skip: int = 0, engine_seed: int | None = None) -> np.ndarray:
    """seed_random_phase<float>(amp, Rng(seed).fork(0)) (rng.hpp:54-67), the
    stream advanced by ``skip`` draws first (OSPR subframe k: skip = k*npix)."""
    a = np.ascontiguousarray(amp, np.float64)
    out = np.empty(a.shape, np.complex64)
    es = fork_seed(seed, 0) if engine_seed is None else engine_seed
    check(lib.hgc_seed_random_phase(_p(a), a.shape[1], a.shape[0], es, skip, _p(out)))
    return out


def mt_jump_state(engine_seed: int, draws: int) -> np.ndarray:
    """std::mt19937_64 state after ``draws`` draws (312 raw words, host jump-ahead)."""
    out = np.empty(312, np.uint64)
    check(lib.hgc_mt_jump_state(engine_seed, draws, _p(out)))
    return out


# ----------------------------------------------------------------- metric
def mse(target: np.ndarray, replay: np.ndarray, cfg: MetricConfig | None = None) -> float:
    """mse() phase-insensitive (metrics.hpp:70-124)."""
    cfg = cfg or MetricConfig()
    if cfg.phase_sensitive:
        raise _lib.HgcUnsupported("mse: phase-sensitive metric is outside the GPU hot path")
    t = np.ascontiguousarray(target, np.float64)
    r = np.ascontiguousarray(replay, np.complex64)
    if t.shape != r.shape:
        raise ValueError("metric: target and replay dimensions mismatch")
    m = None if cfg.mask is None else np.ascontiguousarray(cfg.mask, np.uint8)
    if m is not None and m.shape != t.shape:
        raise ValueError("MetricConfig: mask dimensions mismatch")
    out = C.c_double()
    check(lib.hgc_mse(_p(t), _p(r), _p(m), t.shape[1], t.shape[0], int(cfg.scale_free), C.byref(out)))
    return out.value


def subframe_mse_statistic(per_frame_mse) -> float:  # ospr.hpp:58-64
    v = np.ascontiguousarray(per_frame_mse, np.float64)
    if v.size == 0:
        raise ValueError("subframe_mse_statistic: empty list")
    return float(lib.hgc_subframe_mse_statistic(_p(v), v.size))


# ------------------------------------------------------------------- IFTA
_ALG = {IftaVariant.GS: "gs", IftaVariant.WeightedGS: "wgs", IftaVariant.LiuTaghizadeh: "lt"}


def _ifta_cfg(cfg: IftaConfig) -> _lib.HgcIftaCfg:
    c = _lib.HgcIftaCfg()
    c.variant = int(cfg.variant)
    c.iterations = int(cfg.iterations)
    c.seed = int(cfg.seed) & 0xFFFFFFFFFFFFFFFF
    c.weight_clamp_lo = float(cfg.weight_clamp_lo)
    c.weight_clamp_hi = float(cfg.weight_clamp_hi)
    c.lt_initial_fraction = float(cfg.lt_initial_fraction)
    c.init_phase = int(cfg.init_phase)
    fr = cfg.target.freedoms
    c.freedom_amplitude_outside_roi = int(fr.amplitude_outside_roi)
    c.freedom_phase = int(fr.phase)
    c.freedom_scale = int(fr.scale)
    return c


class _IftaBuffers:
    """Host arrays for one batched IFTA call (inputs + requested outputs)."""

    def __init__(self, cfg: IftaConfig, amps: np.ndarray, seeds, phases=None, init_field=None, init_weights=None,
                 want_hologram=True, want_replay=True, checkpoint=False):
        self.amps = np.ascontiguousarray(amps, np.float64)
        b, ny, nx = self.amps.shape
        K = cfg.iterations
        self.phase = None if phases is None else np.ascontiguousarray(phases, np.float64).reshape(b, ny, nx)
        roi = cfg.target.roi
        self.roi = None if roi is None else np.ascontiguousarray(np.asarray(roi) != 0, np.uint8)
        self.seeds = np.ascontiguousarray(seeds, np.uint64)
        self.init_field = None if init_field is None else np.ascontiguousarray(init_field, np.complex64).reshape(b, ny, nx)
        self.init_weights = None if init_weights is None else np.ascontiguousarray(init_weights, np.float32).reshape(b, ny, nx)
        wide = cfg.slm.levels > 256
        self.levels = np.empty((b, ny, nx), np.uint16 if wide else np.uint8)
        self.hologram = np.empty((b, ny, nx), np.complex64) if want_hologram else None
        self.replay = np.empty((b, ny, nx), np.complex64) if want_replay else None
        self.trace = np.empty((b, K), np.float64)
        self.final_error = np.empty(b, np.float64)
        self.seconds = np.zeros(1, np.float64)
        io = _lib.HgcIftaIo()
        io.amplitude = _p(self.amps)
        io.phase = _p(self.phase)
        io.roi = _p(self.roi)
        io.seeds = _p(self.seeds)
        io.init_field = _p(self.init_field)
        io.init_weights = _p(self.init_weights)
        io.hologram = _p(self.hologram)
        if wide:
            io.levels16 = _p(self.levels)
        else:
            io.levels8 = _p(self.levels)
        io.replay = _p(self.replay)
        io.trace = _p(self.trace)
        io.final_error = _p(self.final_error)
        io.seconds = _p(self.seconds)
        self.profile = np.zeros(4, np.float64)
        io.profile = _p(self.profile)
        io.checkpoint = int(bool(checkpoint))
        self.weights = np.empty((b, ny, nx), np.float32) if checkpoint else None
        io.weights = _p(self.weights)
        self.efficiency = np.zeros(b, np.float64)
        io.efficiency = _p(self.efficiency)
        self.io = io
        self.hologram_gray8 = self.replay_gray8 = self.replay_peak = None

    def want_gray(self, on: bool = True):
        """Also return the runner's hologram.png / replay.png pixels (device-encoded)."""
        b, ny, nx = self.levels.shape
        if on and self.hologram_gray8 is None:
            self.hologram_gray8 = np.empty((b, ny, nx), np.uint8)
            self.replay_gray8 = np.empty((b, ny, nx), np.uint8)
            self.replay_peak = np.empty(b, np.float64)
        self.io.hologram_gray8 = _p(self.hologram_gray8) if on else None
        self.io.replay_gray8 = _p(self.replay_gray8) if on else None
        self.io.replay_peak = _p(self.replay_peak) if on else None


def _check_variant(cfg: IftaConfig, want: IftaVariant | None, name: str):
    if want is not None and cfg.variant != want:
        raise ValueError(f"{name}: config variant mismatch")


def run_ifta_batch(cfg: IftaConfig, amplitudes: np.ndarray, seeds=None, prop: Propagator | None = None,
                   phases=None, init_field=None, init_weights=None, checkpoint=False,
                   want_hologram=True) -> list[RunReport]:
    """B independent targets of one size/SLM/propagation, one launch sequence.
    seeds[b] replaces cfg.seed for target b (default: cfg.seed for all).
    checkpoint: the last iteration also applies the replay-plane constraint;
    each report's `replay` is then the constrained field R_K and `weights`
    the WGS weights W_K — the state a run with init_field / init_weights
    (InitPhase.Given) resumes from (hgc_ifta_io::checkpoint)."""
    amps = np.asarray(amplitudes, np.float64)
    if amps.ndim == 2:
        amps = amps[None]
    b, ny, nx = amps.shape
    if cfg.iterations < 1:
        raise ValueError("IftaConfig: iterations must be >= 1")
    seeds = np.full(b, cfg.seed, np.uint64) if seeds is None else np.asarray(seeds, np.uint64)
    bufs = _IftaBuffers(cfg, amps, seeds, phases, init_field, init_weights, want_hologram=want_hologram,
                        checkpoint=checkpoint)
    keep = []
    slm = _slm(cfg.slm, keep)
    c = _ifta_cfg(cfg)
    fres = _fresnel(prop.params if prop is not None else None)
    check(lib.hgc_ifta_run(C.byref(c), C.byref(slm), fres, nx, ny, b, C.byref(bufs.io)))
    reps = []
    for i in range(b):
        rep = RunReport(algorithm=_ALG[IftaVariant(cfg.variant)], seed=int(seeds[i]))
        rep.hologram = None if bufs.hologram is None else bufs.hologram[i]
        rep.replay = bufs.replay[i]
        rep.levels = bufs.levels[i]
        rep.trace = MetricTrace("mse", [(k + 1, float(v)) for k, v in enumerate(bufs.trace[i])])
        rep.final_error = float(bufs.final_error[i])
        rep.seconds = float(bufs.seconds[0])
        tr, cn, me, ot = (float(v) for v in bufs.profile)  # report.hpp:38-45, whole batched call
        rep.profile = PhaseProfile(transform=tr, constraint=cn, metric=me, other=ot)
        if checkpoint:
            rep.weights = bufs.weights[i]
        rep.efficiency = float(bufs.efficiency[i])
        reps.append(rep)
    return reps


def _run_ifta(cfg: IftaConfig, prop: Propagator | None, want: IftaVariant | None, name: str,
              init_field=None, init_weights=None, checkpoint=False) -> RunReport:
    _check_variant(cfg, want, name)
    cfg.validate()
    if prop is not None and prop.is_fresnel() and (prop.nx, prop.ny) != (cfg.target.width(), cfg.target.height()):
        raise ValueError("Propagator: field size does not match Fresnel phase")
    phases = None if cfg.target.phase is None else np.asarray(cfg.target.phase)[None]
    return run_ifta_batch(cfg, np.asarray(cfg.target.amplitude)[None], [cfg.seed], prop, phases, init_field,
                          init_weights, checkpoint)[0]


def run_gs(cfg: IftaConfig, prop: Propagator | None = None) -> RunReport:  # ifta.hpp:239-244
    return _run_ifta(cfg, prop, IftaVariant.GS, "run_gs")


def run_weighted_gs(cfg: IftaConfig, prop: Propagator | None = None) -> RunReport:  # ifta.hpp:246-251
    return _run_ifta(cfg, prop, IftaVariant.WeightedGS, "run_weighted_gs")


def run_liu_taghizadeh(cfg: IftaConfig, prop: Propagator | None = None) -> RunReport:  # ifta.hpp:253-258
    return _run_ifta(cfg, prop, IftaVariant.LiuTaghizadeh, "run_liu_taghizadeh")


def run_ifta(cfg: IftaConfig, prop: Propagator | None = None, init_field=None, init_weights=None,
             checkpoint=False) -> RunReport:
    """run_ifta<float> (ifta.hpp:260-263); init_field/init_weights serve
    InitPhase.Given (resume from a replay field, e.g. a checkpoint);
    checkpoint=True returns that resume state (see run_ifta_batch)."""
    return _run_ifta(cfg, prop, None, "run_ifta", init_field, init_weights, checkpoint)


def run_ifta_f64(cfg: IftaConfig, prop: Propagator | None = None, init_field=None, init_weights=None) -> RunReport:
    """run_ifta<double> (ifta.hpp:86-235) on the device (hgc_ifta_run_f64,
    SURVEY §8 f4): complex128 hologram / replay, any field size."""
    import time
    cfg.validate()
    amp = np.ascontiguousarray(cfg.target.amplitude, np.float64)
    ny, nx = amp.shape
    if prop is not None and prop.is_fresnel() and (prop.nx, prop.ny) != (nx, ny):
        raise ValueError("Propagator: field size does not match Fresnel phase")
    keep: list = []
    c = _ifta_cfg(cfg)
    slm = _slm(cfg.slm, keep)
    io = _lib.HgcIftaIo64()
    ph = None if cfg.target.phase is None else np.ascontiguousarray(cfg.target.phase, np.float64)
    roi = None if cfg.target.roi is None else np.ascontiguousarray(np.asarray(cfg.target.roi) != 0, np.uint8)
    fi = None if init_field is None else np.ascontiguousarray(init_field, np.complex128)
    wi = None if init_weights is None else np.ascontiguousarray(init_weights, np.float64)
    holo = np.empty((ny, nx), np.complex128)
    rep_f = np.empty((ny, nx), np.complex128)
    lv = np.empty((ny, nx), np.int32)
    tr = np.empty(cfg.iterations, np.float64)
    fe = C.c_double()
    io.amplitude, io.phase, io.roi, io.init_field, io.init_weights = _p(amp), _p(ph), _p(roi), _p(fi), _p(wi)
    io.hologram, io.replay, io.levels, io.trace = _p(holo), _p(rep_f), _p(lv), _p(tr)
    io.final_error = C.addressof(fe)
    prof = np.zeros(4)
    io.profile = _p(prof)
    fr = prop.params if prop is not None and prop.is_fresnel() else None
    t0 = time.perf_counter()
    check(lib.hgc_ifta_run_f64(C.byref(c), C.byref(slm), _fresnel(fr), nx, ny, C.byref(io)))
    rep = RunReport(algorithm=_ALG[IftaVariant(cfg.variant)], seed=int(cfg.seed))
    rep.hologram, rep.replay, rep.levels = holo, rep_f, lv
    rep.trace = MetricTrace("mse", [(k + 1, float(v)) for k, v in enumerate(tr)])
    rep.final_error = fe.value
    rep.seconds = time.perf_counter() - t0
    rep.profile = _profile(prof, rep.seconds)
    return rep


def _profile(p, seconds: float) -> PhaseProfile:
    """RunReport::profile from the library's per-phase device times; other =
    the rest of the call, so total() == seconds (ifta.hpp:231-233)."""
    tr, cn, me = (float(v) for v in p[:3])
    return PhaseProfile(transform=tr, constraint=cn, metric=me, other=max(0.0, seconds - (tr + cn + me)))


def run_ospr_f64(cfg: OsprConfig, keep_frames: bool = True) -> OsprRun:
    """run_ospr_variant<double> (ospr.hpp:68-185) on the device (hgc_ospr_run_f64)."""
    import time
    cfg.validate()
    amp = np.ascontiguousarray(cfg.target.amplitude, np.float64)
    ny, nx = amp.shape
    N = cfg.subframes
    keep: list = []
    c = _ospr_cfg(cfg)
    slm = _slm(cfg.slm, keep)
    roi = None if cfg.target.roi is None else np.ascontiguousarray(np.asarray(cfg.target.roi) != 0, np.uint8)
    frames = np.empty((N, ny, nx), np.complex128) if keep_frames else None
    lv = np.empty((N, ny, nx), np.int32)
    fm, cm = np.empty(N), np.empty(N)
    mi = np.empty((ny, nx))
    rp = np.empty((ny, nx), np.complex128)
    fe = C.c_double()
    io = _lib.HgcOsprIo64()
    io.amplitude, io.roi, io.frames, io.levels = _p(amp), _p(roi), _p(frames), _p(lv)
    io.frame_mse, io.cumulative_mse, io.mean_intensity, io.replay = _p(fm), _p(cm), _p(mi), _p(rp)
    io.final_error = C.addressof(fe)
    prof = np.zeros(4)
    io.profile = _p(prof)
    t0 = time.perf_counter()
    check(lib.hgc_ospr_run_f64(C.byref(c), C.byref(slm), nx, ny, C.byref(io)))
    r = OsprRun()
    r.set = SubframeSet(frames=frames, mean_intensity=mi, per_frame_mse=[float(v) for v in fm], levels=lv)
    rep = RunReport(algorithm="adaptive_ospr" if cfg.variant == OsprVariant.AdaptiveOspr else "ospr",
                    seed=int(cfg.seed))
    rep.trace = MetricTrace("cumulative_mse", [(k + 1, float(v)) for k, v in enumerate(cm)])
    rep.extra_traces = [MetricTrace("frame_mse", [(k + 1, float(v)) for k, v in enumerate(fm)])]
    rep.replay = rp
    rep.hologram = None if frames is None else frames[-1]
    rep.final_error = fe.value
    rep.evaluations = N
    rep.seconds = time.perf_counter() - t0
    rep.profile = _profile(prof, rep.seconds)
    r.report = rep
    return r


# ------------------------------------------------------------------- OSPR
def _ospr_cfg(cfg: OsprConfig) -> _lib.HgcOsprCfg:
    c = _lib.HgcOsprCfg()
    c.variant = int(cfg.variant)
    c.subframes = int(cfg.subframes)
    c.seed = int(cfg.seed) & 0xFFFFFFFFFFFFFFFF
    c.feedback_gain = float(cfg.feedback_gain)
    c.freedom_scale = int(cfg.target.freedoms.scale)
    return c


def run_ospr_batch(cfg: OsprConfig, seeds=None, amplitudes: np.ndarray | None = None,
                   want_frames: bool = True, prop: Propagator | None = None) -> list[OsprRun]:
    """`jobs` independent OSPR runs (one per seed) sharing cfg.target, or one
    target per job when ``amplitudes`` (jobs, ny, nx) is given.  prop: a
    Fresnel Propagator (extension, hgc_ospr_run_fresnel; the reference's
    run_ospr takes a bare FftBackend)."""
    cfg.validate()
    per_job = amplitudes is not None
    amps = np.ascontiguousarray(amplitudes if per_job else cfg.target.amplitude, np.float64)
    seeds = np.asarray([cfg.seed] if seeds is None else seeds, np.uint64)
    jobs = len(seeds)
    ny, nx = amps.shape[-2:]
    N = cfg.subframes
    wide = cfg.slm.levels > 256
    lv = np.empty((jobs, N, ny, nx), np.uint16 if wide else np.uint8)
    frames = np.empty((jobs, N, ny, nx), np.complex64) if want_frames else None
    fm = np.empty((jobs, N), np.float64)
    cm = np.empty((jobs, N), np.float64)
    mi = np.empty((jobs, ny, nx), np.float64)
    rp = np.empty((jobs, ny, nx), np.complex64)
    fe = np.empty(jobs, np.float64)
    secs = np.zeros(1, np.float64)
    roi = None if cfg.target.roi is None else np.ascontiguousarray(np.asarray(cfg.target.roi) != 0, np.uint8)
    io = _lib.HgcOsprIo()
    io.amplitude = _p(amps)
    io.per_job_target = int(per_job)
    io.roi = _p(roi)
    io.seeds = _p(seeds)
    if wide:
        io.levels16 = _p(lv)
    else:
        io.levels8 = _p(lv)
    io.frames = _p(frames)
    io.frame_mse, io.cumulative_mse = _p(fm), _p(cm)
    io.mean_intensity, io.replay, io.final_error, io.seconds = _p(mi), _p(rp), _p(fe), _p(secs)
    prof = np.zeros(4)
    io.profile = _p(prof)
    keep = []
    slm = _slm(cfg.slm, keep)
    c = _ospr_cfg(cfg)
    fr = prop.params if prop is not None and prop.is_fresnel() else None
    if fr is not None and (prop.nx, prop.ny) != (nx, ny):
        raise ValueError("Propagator: field size does not match Fresnel phase")
    check(lib.hgc_ospr_run_fresnel(C.byref(c), C.byref(slm), _fresnel(fr), nx, ny, jobs, C.byref(io)))
    runs = []
    alg = "adaptive_ospr" if cfg.variant == OsprVariant.AdaptiveOspr else "ospr"
    for j in range(jobs):
        r = OsprRun()
        r.set = SubframeSet(frames=None if frames is None else frames[j], mean_intensity=mi[j],
                            per_frame_mse=[float(v) for v in fm[j]], levels=lv[j])
        rep = RunReport(algorithm=alg, seed=int(seeds[j]))
        rep.trace = MetricTrace("cumulative_mse", [(k + 1, float(v)) for k, v in enumerate(cm[j])])
        rep.extra_traces = [MetricTrace("frame_mse", [(k + 1, float(v)) for k, v in enumerate(fm[j])])]
        rep.hologram = None if frames is None else frames[j, -1]
        rep.levels = lv[j, -1]
        rep.replay = rp[j]
        rep.final_error = float(fe[j])
        rep.evaluations = N
        rep.seconds = float(secs[0])
        rep.profile = _profile(prof, rep.seconds)  # whole batched call
        r.report = rep
        runs.append(r)
    return runs


def run_ospr(cfg: OsprConfig, prop: Propagator | None = None) -> OsprRun:  # ospr.hpp:168-173
    if cfg.variant != OsprVariant.Ospr:
        raise ValueError("run_ospr: config variant mismatch")
    return run_ospr_batch(cfg, prop=prop)[0]


def run_adaptive_ospr(cfg: OsprConfig, prop: Propagator | None = None) -> OsprRun:  # ospr.hpp:175-180
    if cfg.variant != OsprVariant.AdaptiveOspr:
        raise ValueError("run_adaptive_ospr: config variant mismatch")
    return run_ospr_batch(cfg, prop=prop)[0]


def run_ospr_variant(cfg: OsprConfig, prop: Propagator | None = None) -> OsprRun:  # ospr.hpp:182-185
    return run_ospr_batch(cfg, prop=prop)[0]


# -------------------------------------------------- device-resident plans
class _CudaArray:
    """__cuda_array_interface__ view of a library-owned device buffer."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


class IftaPlan:
    """Resident batched IFTA run: upload once, execute many times on a stream."""

    def __init__(self, cfg: IftaConfig, nx: int, ny: int, batch: int, prop: Propagator | None = None):
        cfg.slm.validate()
        self.cfg, self.nx, self.ny, self.batch = cfg, nx, ny, batch
        self._keep = []
        self._c = _ifta_cfg(cfg)
        self._slm = _slm(cfg.slm, self._keep)
        self._fres = None if prop is None or prop.params is None else _lib.HgcFresnel(
            prop.params.wavelength, prop.params.distance, prop.params.pixel_pitch_x, prop.params.pixel_pitch_y)
        h = C.c_void_p()
        check(lib.hgc_ifta_plan_create(C.byref(h), C.byref(self._c), C.byref(self._slm),
                                       None if self._fres is None else C.byref(self._fres), nx, ny, batch))
        self._h = h
        self._bufs = None

    def upload(self, amplitudes: np.ndarray, seeds=None, phases=None, init_field=None, init_weights=None):
        amps = np.asarray(amplitudes, np.float64).reshape(self.batch, self.ny, self.nx)
        seeds = np.full(self.batch, self.cfg.seed, np.uint64) if seeds is None else np.asarray(seeds, np.uint64)
        self._bufs = _IftaBuffers(self.cfg, amps, seeds, phases, init_field, init_weights)
        check(lib.hgc_ifta_plan_upload(self._h, C.byref(self._bufs.io)))

    def execute(self, stream: int | None = None):
        check(lib.hgc_ifta_plan_execute(self._h, stream))

    def download(self, gray: bool = False):
        """Copy results back; gray=True adds hologram_gray8 / replay_gray8 /
        replay_peak (write_hologram_png / write_replay_png pixels)."""
        self._bufs.want_gray(gray)
        check(lib.hgc_ifta_plan_download(self._h, C.byref(self._bufs.io)))
        return self._bufs

    def launches(self) -> int:
        return int(lib.hgc_ifta_plan_launches(self._h))

    def set_kernel_timing(self, on: bool = True):
        """Record CUDA events around the passes inside the plan's graph (call
        before the first execute); read them with kernel_times()."""
        check(lib.hgc_ifta_plan_set_kernel_timing(self._h, int(on)))

    def kernel_times(self) -> dict:
        """Average row / column pass device ms of the last execute, measured
        inside its graph (iterations 1..K-1 of the first target group)."""
        r, c, n = C.c_double(), C.c_double(), C.c_int()
        check(lib.hgc_ifta_plan_kernel_times(self._h, C.byref(r), C.byref(c), C.byref(n)))
        return {"row": r.value, "col": c.value, "iterations": n.value}

    def profile(self, reps: int = 5) -> dict:
        """Per-kernel device ms: seed, fused row pass, fused column pass."""
        s, r, c = C.c_double(), C.c_double(), C.c_double()
        check(lib.hgc_ifta_plan_profile(self._h, reps, C.byref(s), C.byref(r), C.byref(c)))
        return {"seed": s.value, "row": r.value, "col": c.value}

    def device_arrays(self):
        """(replay field, levels, trace) as __cuda_array_interface__ objects."""
        f, lv, tr = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(lib.hgc_ifta_plan_device_ptrs(self._h, C.byref(f), C.byref(lv), C.byref(tr)))
        b, ny, nx = self.batch, self.ny, self.nx
        lt = "<u2" if self.cfg.slm.levels > 256 else "|u1"
        return (_CudaArray(f.value, (b, ny, nx, 2), "<f4"), _CudaArray(lv.value, (b, ny, nx), lt),
                _CudaArray(tr.value, (b, self.cfg.iterations), "<f8"))

    def close(self):
        if getattr(self, "_h", None):
            lib.hgc_ifta_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


class OsprPlan:
    """Resident batched OSPR run over `jobs` seeds (shared or per-job target)."""

    def __init__(self, cfg: OsprConfig, nx: int, ny: int, jobs: int, per_job_target: bool = False):
        cfg.slm.validate()
        self.cfg, self.nx, self.ny, self.jobs, self.per_job = cfg, nx, ny, jobs, per_job_target
        self._nf = cfg.subframes
        self._keep = []
        self._c = _ospr_cfg(cfg)
        self._slm = _slm(cfg.slm, self._keep)
        h = C.c_void_p()
        check(lib.hgc_ospr_plan_create(C.byref(h), C.byref(self._c), C.byref(self._slm), nx, ny, jobs,
                                       int(per_job_target)))
        self._h = h
        self._io = None

    def upload(self, amplitude: np.ndarray, seeds=None, roi=None):
        self._amp = np.ascontiguousarray(amplitude, np.float64)
        self._seeds = np.asarray([self.cfg.seed] * self.jobs if seeds is None else seeds, np.uint64)
        self._roi = None if roi is None else np.ascontiguousarray(np.asarray(roi) != 0, np.uint8)
        io = _lib.HgcOsprIo()
        io.amplitude, io.per_job_target, io.roi, io.seeds = _p(self._amp), int(self.per_job), _p(self._roi), \
            _p(self._seeds)
        self._io = io
        check(lib.hgc_ospr_plan_upload(self._h, C.byref(io)))

    def execute(self, stream: int | None = None):
        check(lib.hgc_ospr_plan_execute(self._h, stream))

    def download(self, frames: bool = False, gray: bool = False, bits: bool = False):
        """bits=True (2-level SLMs) adds "levels1": the frames as bit-planes
        [jobs][N][npix/8], bit (i & 7) of byte i >> 3 (np.packbits little)."""
        N = self._nf
        jobs, ny, nx = self.jobs, self.ny, self.nx
        wide = self.cfg.slm.levels > 256
        out = {"levels": np.empty((jobs, N, ny, nx), np.uint16 if wide else np.uint8),
               "frame_mse": np.empty((jobs, N)), "cumulative_mse": np.empty((jobs, N)),
               "mean_intensity": np.empty((jobs, ny, nx)), "final_error": np.empty(jobs)}
        io = _lib.HgcOsprIo()
        if wide:
            io.levels16 = _p(out["levels"])
        else:
            io.levels8 = _p(out["levels"])
        if frames:
            out["frames"] = np.empty((jobs, N, ny, nx), np.complex64)
            io.frames = _p(out["frames"])
        io.frame_mse, io.cumulative_mse = _p(out["frame_mse"]), _p(out["cumulative_mse"])
        io.mean_intensity, io.final_error = _p(out["mean_intensity"]), _p(out["final_error"])
        if bits:
            out["levels1"] = np.empty((jobs, N, ny * nx // 8), np.uint8)
            io.levels1 = _p(out["levels1"])
        if gray:  # device-encoded hologram.png per frame / replay.png pixels
            out["frames_gray8"] = np.empty((jobs, N, ny, nx), np.uint8)
            out["replay_gray8"] = np.empty((jobs, ny, nx), np.uint8)
            out["replay_peak"] = np.empty(jobs)
            io.frames_gray8, io.replay_gray8 = _p(out["frames_gray8"]), _p(out["replay_gray8"])
            io.replay_peak = _p(out["replay_peak"])
        check(lib.hgc_ospr_plan_download(self._h, C.byref(io)))
        return out

    def launches(self) -> int:
        return int(lib.hgc_ospr_plan_launches(self._h))

    def profile(self, reps: int = 5) -> dict:
        """Per-kernel device ms of one subframe: seed, col_inv, row, col_acc."""
        v = [C.c_double() for _ in range(4)]
        check(lib.hgc_ospr_plan_profile(self._h, reps, *[C.byref(x) for x in v]))
        return dict(zip(("seed", "col_inv", "row", "col_acc"), (x.value for x in v)))

    def device_arrays(self):
        lv, tr, S = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(lib.hgc_ospr_plan_device_ptrs(self._h, C.byref(lv), C.byref(tr), C.byref(S)))
        N = self._nf
        lt = "<u2" if self.cfg.slm.levels > 256 else "|u1"
        return (_CudaArray(lv.value, (self.jobs, N, self.ny, self.nx), lt),
                _CudaArray(tr.value, (self.jobs, N, 2), "<f8"),
                _CudaArray(S.value, (self.jobs, self.ny, self.nx), "<f4"))

    def close(self):
        if getattr(self, "_h", None):
            lib.hgc_ospr_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


class OsprBlockPlan(OsprPlan):
    """Global subframes [first, first + count) of ONE plain OSPR job (SURVEY
    §8 e2): the stream starts first*npix draws into Rng(seed).fork(0) by
    jump-ahead.  After execute, all-gather every block's ``block_sum()`` in
    block order and call ``finish`` to get the cumulative MSEs and the job's
    mean intensity (hgc_ospr_block_*)."""

    def __init__(self, cfg: OsprConfig, nx: int, ny: int, first: int, count: int):
        cfg.slm.validate()
        self.cfg, self.nx, self.ny, self.jobs, self.per_job = cfg, nx, ny, 1, False
        self.first, self.count, self._nf = first, count, count
        self._keep = []
        self._c = _ospr_cfg(cfg)
        self._slm = _slm(cfg.slm, self._keep)
        h = C.c_void_p()
        check(lib.hgc_ospr_block_plan_create(C.byref(h), C.byref(self._c), C.byref(self._slm), nx, ny, first, count))
        self._h = h
        self._io = None

    def block_sum(self) -> "_CudaArray":
        ptr, n = C.c_void_p(), C.c_size_t()
        check(lib.hgc_ospr_block_sum(self._h, C.byref(ptr), C.byref(n)))
        return _CudaArray(ptr.value, (n.value,), "<f4")

    def finish(self, gathered_ptr: int, nblocks: int, index: int, stream: int | None = None):
        check(lib.hgc_ospr_block_finish(self._h, gathered_ptr, nblocks, index, stream))


def device_count() -> int:
    n = C.c_int(0)
    check(lib.hgc_device_count(C.byref(n)))
    return n.value


def set_device(dev: int) -> None:
    check(lib.hgc_set_device(dev))
