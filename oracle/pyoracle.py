"""ctypes front end to the CPU oracle — TEST INFRASTRUCTURE ONLY.

Two back ends with one interface:

* ``Oracle("restatement")`` — oracle/libhgoracle.so, the plain-C restatement
  (oracle/hg_oracle.c) of the reference's IFTA/OSPR path;
* ``Oracle("reference")``   — oracle/_ref/libhgref.so, the reference's own
  unmodified headers compiled here (oracle/ref_shim.cpp).

Only tests/, ``__graft_entry__.smoke()`` and bench.py (its cpu_baseline and
``--impl reference`` legs) import this module, and only as the checker or the
timed CPU baseline.  The product package never imports it.

Duck-typed inputs: ``slm`` is any object with the attributes of
``hologen::SlmSpec`` (mode, levels, min_arg, max_arg, full_circle, min_amp,
max_amp, illumination) — e.g. ``paper_2008_12214_b200.SlmSpec``.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "restatement": os.path.join(HERE, "libhgoracle.so"),
    "reference": os.path.join(HERE, "_ref", "libhgref.so"),
}


class HgoSlm(C.Structure):
    _fields_ = [
        ("mode", C.c_int),
        ("levels", C.c_int),
        ("min_arg", C.c_double),
        ("max_arg", C.c_double),
        ("full_circle", C.c_int),
        ("min_amp", C.c_double),
        ("max_amp", C.c_double),
        ("illum", C.c_void_p),
    ]


class HgoIftaCfg(C.Structure):
    _fields_ = [
        ("variant", C.c_int),
        ("iterations", C.c_int),
        ("seed", C.c_uint64),
        ("clamp_lo", C.c_double),
        ("clamp_hi", C.c_double),
        ("lt_initial_fraction", C.c_double),
        ("init_phase", C.c_int),
        ("amp_outside_roi", C.c_int),
        ("phase_freedom", C.c_int),
        ("scale_freedom", C.c_int),
        ("fresnel", C.c_int),
        ("wavelength", C.c_double),
        ("distance", C.c_double),
        ("pitch_x", C.c_double),
        ("pitch_y", C.c_double),
        ("snapshot_iter", C.c_int),
    ]


def build():
    """Build the oracle libraries (make -C oracle)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def available(kind: str) -> bool:
    return os.path.exists(LIBS[kind])


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _slm(slm, keep):
    s = HgoSlm()
    m = getattr(slm, "mode", 1)
    s.mode = (1 if m.lower().endswith("phase") else 0) if isinstance(m, str) else int(m)
    s.levels = int(slm.levels)
    s.min_arg = float(slm.min_arg)
    s.max_arg = float(slm.max_arg)
    s.full_circle = int(bool(slm.full_circle))
    s.min_amp = float(slm.min_amp)
    s.max_amp = float(slm.max_amp)
    il = getattr(slm, "illumination", None)
    if il is not None:
        il = np.ascontiguousarray(il, dtype=np.complex128)
        keep.append(il)
        s.illum = il.ctypes.data
    else:
        s.illum = None
    return s


@dataclass
class IftaResult:
    hologram: np.ndarray  # complex64 (ny, nx)
    replay: np.ndarray  # complex64 (ny, nx)
    levels: np.ndarray  # int32 (ny, nx)
    trace: np.ndarray  # float64 (K,)
    snap_r: np.ndarray | None = None
    snap_w: np.ndarray | None = None
    seconds: float = 0.0
    profile: tuple | None = None  # (transform, constraint, metric, other) seconds, reference only


@dataclass
class OsprResult:
    levels: np.ndarray  # int32 (N, ny, nx)
    frames: np.ndarray | None  # complex64 (N, ny, nx)
    frame_mse: np.ndarray
    cumulative_mse: np.ndarray
    mean_intensity: np.ndarray  # float64 (ny, nx)
    replay: np.ndarray  # complex64 (ny, nx)
    seconds: float = 0.0


class Oracle:
    def __init__(self, kind: str = "restatement"):
        path = LIBS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run make -C oracle)")
        self.kind = kind
        self.lib = L = C.CDLL(path)
        self.pre = "hgo_" if kind == "restatement" else "hgr_"
        vp, i, u64, d, sz = C.c_void_p, C.c_int, C.c_uint64, C.c_double, C.c_size_t
        self._f = {}

        def fn(name, res, args):
            f = getattr(L, self.pre + name)
            f.restype = res
            f.argtypes = args
            self._f[name] = f

        fn("mix64", u64, [u64])
        fn("fork_seed", u64, [u64, u64])
        fn("mt_draws", None, [u64, u64, sz, vp])
        fn("quant_states", None, [C.POINTER(HgoSlm), vp])
        fn("fresnel_q", None if kind == "restatement" else i, [i, i, d, d, d, d, vp])
        fn("subframe_mse_statistic", d, [vp, i])
        if kind == "restatement":
            fn("seed_random_phase_seeded", None, [vp, sz, u64, u64, vp])
            fn("quantise", i, [C.POINTER(HgoSlm), i, i, vp, vp])
            fn("fft2d", None, [i, i, i, vp, vp])
            fn("fft2d_d", None, [i, i, i, vp, vp])
            fn("fft2d_fastf", None, [i, i, i, vp, vp])
            fn("mse", d, [vp, vp, vp, sz, i])
            fn("ifta_run", i, [C.POINTER(HgoIftaCfg), C.POINTER(HgoSlm), i, i, vp, vp, vp, vp, vp,
                               vp, vp, vp, vp, vp, vp])
            fn("ifta_run_snaps", i, [C.POINTER(HgoIftaCfg), C.POINTER(HgoSlm), i, i, vp, vp, vp, vp, vp,
                                     vp, vp, i, vp, vp, vp, vp])
            fn("ospr_run", i, [i, i, u64, d, C.POINTER(HgoSlm), i, i, vp, vp, i, vp, vp, vp, vp, vp, vp])
        else:
            fn("last_error", C.c_char_p, [])
            fn("set_fast_fft", None, [i])
            fn("seed_random_phase", i, [vp, i, i, u64, u64, vp])
            fn("quantise", i, [C.POINTER(HgoSlm), i, i, vp, vp])
            fn("fft", i, [i, i, i, i, vp, vp])
            fn("fft_d", i, [i, i, i, i, vp, vp])
            fn("mse", i, [vp, vp, vp, i, i, i, vp])
            fn("smooth_blobs", None, [i, i, vp])
            fn("normalize", i, [vp, i, i, i])
            fn("ifta_run", i, [C.POINTER(HgoIftaCfg), C.POINTER(HgoSlm), i, i, vp, vp, vp, vp, vp,
                               vp, vp, vp])
            fn("ospr_run", i, [i, i, u64, d, C.POINTER(HgoSlm), i, i, vp, vp, i, vp, vp, vp, vp, vp, vp,
                               vp])
            fn("ifta_run_d", i, [C.POINTER(HgoIftaCfg), C.POINTER(HgoSlm), i, i, vp, vp, vp, vp, vp, vp, vp])
            fn("ospr_run_d", i, [i, i, u64, d, C.POINTER(HgoSlm), i, i, vp, vp, i, vp, vp, vp, vp])

    # ------------------------------------------------------------ helpers
    def _check(self, rc):
        if rc != 0:
            msg = self._f["last_error"]().decode() if self.kind == "reference" else "invalid input"
            raise ValueError(msg)

    def set_fast_fft(self, on: bool):
        if self.kind == "reference":
            self._f["set_fast_fft"](int(on))

    # ---------------------------------------------------------------- rng
    def mix64(self, z: int) -> int:
        return self._f["mix64"](z)

    def fork_seed(self, seed: int, stream: int = 0) -> int:
        return self._f["fork_seed"](seed, stream)

    def mt_draws(self, seed: int, n: int, skip: int = 0) -> np.ndarray:
        out = np.empty(n, np.uint64)
        self._f["mt_draws"](seed, skip, n, _p(out))
        return out

    def seed_random_phase(self, amp: np.ndarray, seed: int, skip: int = 0) -> np.ndarray:
        amp = np.ascontiguousarray(amp, np.float64)
        out = np.empty(amp.shape, np.complex64)
        if self.kind == "restatement":
            self._f["seed_random_phase_seeded"](_p(amp), amp.size, seed, skip, _p(out))
        else:
            ny, nx = amp.shape
            self._check(self._f["seed_random_phase"](_p(amp), nx, ny, seed, skip, _p(out)))
        return out

    # ---------------------------------------------------------- quantiser
    def quantise(self, slm, field: np.ndarray):
        keep = []
        s = _slm(slm, keep)
        f = np.ascontiguousarray(field, np.complex64).copy()
        ny, nx = f.shape
        lv = np.empty((ny, nx), np.int32)
        self._check(self._f["quantise"](C.byref(s), nx, ny, _p(f), _p(lv)))
        return f, lv

    def quant_states(self, slm) -> np.ndarray:
        keep = []
        s = _slm(slm, keep)
        out = np.empty(int(slm.levels), np.complex64)
        self._f["quant_states"](C.byref(s), _p(out))
        return out

    def fresnel_q(self, nx, ny, wavelength, distance, px, py) -> np.ndarray:
        q = np.empty((ny, nx), np.complex64)
        self._f["fresnel_q"](nx, ny, wavelength, distance, px, py, _p(q))
        return q

    # ---------------------------------------------------------------- fft
    def fft2(self, x: np.ndarray, sign: int, naive: bool = False, fast: bool = False) -> np.ndarray:
        """Unitary 2-D DFT, sign -1 forward / +1 inverse (fft.hpp:17-27)."""
        x = np.ascontiguousarray(x)
        ny, nx = x.shape
        dbl = x.dtype == np.complex128
        out = np.empty_like(x)
        if self.kind == "restatement":
            if naive:
                raise ValueError("naive DFT lives in the reference (fft.hpp:32-77)")
            name = "fft2d_d" if dbl else ("fft2d_fastf" if fast else "fft2d")
            self._f[name](nx, ny, sign, _p(x), _p(out))
        else:
            self._check(self._f["fft_d" if dbl else "fft"](nx, ny, sign, int(naive), _p(x), _p(out)))
        return out

    # ---------------------------------------------------------------- mse
    def mse(self, target, replay, mask=None, scale_free=False) -> float:
        t = np.ascontiguousarray(target, np.float64)
        r = np.ascontiguousarray(replay, np.complex64)
        m = None if mask is None else np.ascontiguousarray(mask, np.uint8)
        if self.kind == "restatement":
            return self._f["mse"](_p(t), _p(r), _p(m), t.size, int(scale_free))
        out = C.c_double()
        ny, nx = t.shape
        self._check(self._f["mse"](_p(t), _p(r), _p(m), nx, ny, int(scale_free), C.byref(out)))
        return out.value

    def subframe_mse_statistic(self, v) -> float:
        v = np.ascontiguousarray(v, np.float64)
        return self._f["subframe_mse_statistic"](_p(v), v.size)

    # ------------------------------------------------- reference patterns
    def smooth_blobs(self, w, h) -> np.ndarray:
        out = np.empty((h, w), np.float64)
        self._f["smooth_blobs"](w, h, _p(out))
        return out

    def normalize(self, img, unit_energy=True) -> np.ndarray:
        out = np.ascontiguousarray(img, np.float64).copy()
        h, w = out.shape
        self._check(self._f["normalize"](_p(out), w, h, int(unit_energy)))
        return out

    # --------------------------------------------------------------- ifta
    def ifta(self, amp, slm, iterations, seed=0, variant="gs", phase_turns=None, roi=None,
             clamp=(0.1, 10.0), lt_initial_fraction=0.1, init_phase="auto",
             amp_outside_roi=False, phase_freedom=True, scale_freedom=False, fresnel=None,
             init_field=None, init_weights=None, snapshot_iter=0) -> IftaResult:
        keep = []
        amp = np.ascontiguousarray(amp, np.float64)
        ny, nx = amp.shape
        c = HgoIftaCfg()
        c.variant = {"gs": 0, "wgs": 1, "lt": 2}[variant]
        c.iterations = iterations
        c.seed = seed
        c.clamp_lo, c.clamp_hi = clamp
        c.lt_initial_fraction = lt_initial_fraction
        c.init_phase = {"auto": 0, "random": 1, "flat": 2, "given": 3}[init_phase]
        c.amp_outside_roi = int(amp_outside_roi)
        c.phase_freedom = int(phase_freedom)
        c.scale_freedom = int(scale_freedom)
        if fresnel is not None:
            c.fresnel = 1
            c.wavelength, c.distance, c.pitch_x, c.pitch_y = fresnel
        c.snapshot_iter = snapshot_iter
        s = _slm(slm, keep)
        ph = None if phase_turns is None else np.ascontiguousarray(phase_turns, np.float64)
        rm = None if roi is None else np.ascontiguousarray(roi, np.uint8)
        holo = np.empty((ny, nx), np.complex64)
        rep = np.empty((ny, nx), np.complex64)
        lv = np.empty((ny, nx), np.int32)
        tr = np.empty(iterations, np.float64)
        if self.kind == "restatement":
            fi = None if init_field is None else np.ascontiguousarray(init_field, np.complex64)
            wi = None if init_weights is None else np.ascontiguousarray(init_weights, np.float64)
            sr = np.empty((ny, nx), np.complex64) if snapshot_iter else None
            sw = np.empty((ny, nx), np.float64) if snapshot_iter and variant == "wgs" else None
            rc = self._f["ifta_run"](C.byref(c), C.byref(s), nx, ny, _p(amp), _p(ph), _p(rm), _p(fi),
                                     _p(wi), _p(holo), _p(rep), _p(lv), _p(tr), _p(sr), _p(sw))
            self._check(rc)
            return IftaResult(holo, rep, lv, tr, sr, sw)
        if init_field is not None or snapshot_iter:
            raise ValueError("snapshots / given init are restatement-only hooks")
        tm = np.zeros(5, np.float64)  # RunReport seconds, profile transform/constraint/metric/other
        self._check(self._f["ifta_run"](C.byref(c), C.byref(s), nx, ny, _p(amp), _p(ph), _p(rm),
                                        _p(holo), _p(rep), _p(lv), _p(tr), _p(tm)))
        return IftaResult(holo, rep, lv, tr, seconds=float(tm[0]), profile=tuple(float(v) for v in tm[1:]))

    def ifta_snaps(self, amp, slm, iterations, snap_iters, seed=0, variant="gs", clamp=(0.1, 10.0),
                   fresnel=None, scale_freedom=False, roi=None, amp_outside_roi=False, lt_initial_fraction=0.1):
        """Restatement run with snapshots at the start of each iteration k in
        snap_iters: returns (IftaResult, {k: (R_{k-1}, W_{k-1} or None, levels_k)}).
        Test hook for the lock-step parity protocol."""
        if self.kind != "restatement":
            raise ValueError("snapshots are a restatement-only hook")
        keep = []
        amp = np.ascontiguousarray(amp, np.float64)
        ny, nx = amp.shape
        c = HgoIftaCfg()
        c.variant = {"gs": 0, "wgs": 1, "lt": 2}[variant]
        c.iterations = iterations
        c.seed = seed
        c.clamp_lo, c.clamp_hi = clamp
        c.lt_initial_fraction = lt_initial_fraction
        c.phase_freedom = 1
        c.scale_freedom = int(scale_freedom)
        c.amp_outside_roi = int(amp_outside_roi)
        rm = None if roi is None else np.ascontiguousarray(roi, np.uint8)
        if fresnel is not None:
            c.fresnel = 1
            c.wavelength, c.distance, c.pitch_x, c.pitch_y = fresnel
        s = _slm(slm, keep)
        ks = np.ascontiguousarray(sorted(set(int(k) for k in snap_iters)), np.int32)
        m = len(ks)
        sr = np.empty((m, ny, nx), np.complex64)
        sw = np.empty((m, ny, nx), np.float64) if variant == "wgs" else None
        sl = np.empty((m, ny, nx), np.int32)
        holo = np.empty((ny, nx), np.complex64)
        rep = np.empty((ny, nx), np.complex64)
        lv = np.empty((ny, nx), np.int32)
        tr = np.empty(iterations, np.float64)
        self._check(self._f["ifta_run_snaps"](C.byref(c), C.byref(s), nx, ny, _p(amp), None, _p(rm), _p(holo),
                                              _p(rep), _p(lv), _p(tr), m, _p(ks), _p(sr), _p(sw), _p(sl)))
        snaps = {int(k): (sr[j], None if sw is None else sw[j], sl[j]) for j, k in enumerate(ks)}
        return IftaResult(holo, rep, lv, tr), snaps

    def ifta64(self, amp, slm, iterations, seed=0, variant="gs", phase_turns=None, roi=None,
               clamp=(0.1, 10.0), lt_initial_fraction=0.1, init_phase="auto", amp_outside_roi=False,
               phase_freedom=True, scale_freedom=False, fresnel=None) -> IftaResult:
        """run_ifta<double> of the compiled reference (kind == "reference" only)."""
        keep = []
        amp = np.ascontiguousarray(amp, np.float64)
        ny, nx = amp.shape
        c = HgoIftaCfg()
        c.variant = {"gs": 0, "wgs": 1, "lt": 2}[variant]
        c.iterations = iterations
        c.seed = seed
        c.clamp_lo, c.clamp_hi = clamp
        c.lt_initial_fraction = lt_initial_fraction
        c.init_phase = {"auto": 0, "random": 1, "flat": 2}[init_phase]
        c.amp_outside_roi = int(amp_outside_roi)
        c.phase_freedom = int(phase_freedom)
        c.scale_freedom = int(scale_freedom)
        if fresnel is not None:
            c.fresnel = 1
            c.wavelength, c.distance, c.pitch_x, c.pitch_y = fresnel
        s = _slm(slm, keep)
        ph = None if phase_turns is None else np.ascontiguousarray(phase_turns, np.float64)
        rm = None if roi is None else np.ascontiguousarray(roi, np.uint8)
        holo = np.empty((ny, nx), np.complex128)
        rep = np.empty((ny, nx), np.complex128)
        lv = np.empty((ny, nx), np.int32)
        tr = np.empty(iterations, np.float64)
        self._check(self._f["ifta_run_d"](C.byref(c), C.byref(s), nx, ny, _p(amp), _p(ph), _p(rm), _p(holo),
                                          _p(rep), _p(lv), _p(tr)))
        return IftaResult(holo, rep, lv, tr)

    def ospr64(self, target, slm, subframes, seed=0, adaptive=False, gain=1.0, roi=None,
               scale_free=False) -> OsprResult:
        """run_ospr_variant<double> of the compiled reference (kind == "reference" only)."""
        keep = []
        t = np.ascontiguousarray(target, np.float64)
        ny, nx = t.shape
        s = _slm(slm, keep)
        rm = None if roi is None else np.ascontiguousarray(roi, np.uint8)
        lv = np.empty((subframes, ny, nx), np.int32)
        fm = np.empty(subframes, np.float64)
        cm = np.empty(subframes, np.float64)
        mi = np.empty((ny, nx), np.float64)
        self._check(self._f["ospr_run_d"](int(adaptive), subframes, seed, gain, C.byref(s), nx, ny, _p(t), _p(rm),
                                          int(scale_free), _p(lv), _p(fm), _p(cm), _p(mi)))
        return OsprResult(lv, None, fm, cm, mi, None)

    # --------------------------------------------------------------- ospr
    def ospr(self, target, slm, subframes, seed=0, adaptive=False, gain=1.0, roi=None,
             scale_free=False, keep_frames=False) -> OsprResult:
        keep = []
        t = np.ascontiguousarray(target, np.float64)
        ny, nx = t.shape
        s = _slm(slm, keep)
        rm = None if roi is None else np.ascontiguousarray(roi, np.uint8)
        lv = np.empty((subframes, ny, nx), np.int32)
        fr = np.empty((subframes, ny, nx), np.complex64) if keep_frames else None
        fm = np.empty(subframes, np.float64)
        cm = np.empty(subframes, np.float64)
        mi = np.empty((ny, nx), np.float64)
        rp = np.empty((ny, nx), np.complex64)
        args = [int(adaptive), subframes, seed, gain, C.byref(s), nx, ny, _p(t), _p(rm),
                int(scale_free), _p(lv), _p(fr), _p(fm), _p(cm), _p(mi), _p(rp)]
        secs = C.c_double()
        if self.kind == "reference":
            args.append(C.byref(secs))
        self._check(self._f["ospr_run"](*args))
        return OsprResult(lv, fr, fm, cm, mi, rp, secs.value)
