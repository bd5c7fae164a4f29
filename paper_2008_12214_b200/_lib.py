"""ctypes binding of the C ABI in include/hologen_b200.h.

Loads the in-tree ``libhologen_b200.so`` (built by ``build.py`` /
``__graft_entry__.build()``).  There is no fallback: if the library is
missing the import fails, and every call that needs a GPU raises when none is
present.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HG_LIB") or os.path.join(_HERE, "libhologen_b200.so")  # HG_LIB: tuning builds
HEADER_PATH = os.path.join(os.path.dirname(_HERE), "include", "hologen_b200.h")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build the sm_100a library first "
        "(python -c 'import __graft_entry__ as g; g.build()' or python paper_2008_12214_b200/build.py)")

lib = C.CDLL(LIB_PATH)

HGC_OK, HGC_EINVAL, HGC_ECUDA, HGC_EUNSUPPORTED, HGC_EIO = 0, 1, 2, 3, 4


class HgcError(RuntimeError):
    """Device/runtime failure (std::runtime_error in the reference)."""


class HgcUnsupported(HgcError):
    """Valid for the reference but outside the GPU path (no CPU fallback)."""


class HgcIOError(RuntimeError):
    """File / format error (std::runtime_error from io.cpp in the reference)."""


class HgcSlm(C.Structure):
    _fields_ = [("mode", C.c_int), ("levels", C.c_int), ("min_arg", C.c_double), ("max_arg", C.c_double),
                ("full_circle", C.c_int), ("min_amp", C.c_double), ("max_amp", C.c_double),
                ("illumination", C.c_void_p)]


class HgcFresnel(C.Structure):
    _fields_ = [("wavelength", C.c_double), ("distance", C.c_double), ("pixel_pitch_x", C.c_double),
                ("pixel_pitch_y", C.c_double)]


class HgcIftaCfg(C.Structure):
    _fields_ = [("variant", C.c_int), ("iterations", C.c_int), ("seed", C.c_uint64),
                ("weight_clamp_lo", C.c_double), ("weight_clamp_hi", C.c_double),
                ("lt_initial_fraction", C.c_double), ("init_phase", C.c_int),
                ("freedom_amplitude_outside_roi", C.c_int), ("freedom_phase", C.c_int),
                ("freedom_scale", C.c_int)]


class HgcIftaIo(C.Structure):
    _fields_ = [("amplitude", C.c_void_p), ("phase", C.c_void_p), ("roi", C.c_void_p), ("seeds", C.c_void_p),
                ("init_field", C.c_void_p), ("init_weights", C.c_void_p), ("hologram", C.c_void_p),
                ("levels8", C.c_void_p), ("levels16", C.c_void_p), ("replay", C.c_void_p),
                ("trace", C.c_void_p), ("final_error", C.c_void_p), ("seconds", C.c_void_p),
                ("fresnel_q", C.c_void_p), ("hologram_gray8", C.c_void_p), ("replay_gray8", C.c_void_p),
                ("replay_peak", C.c_void_p), ("levels1", C.c_void_p), ("checkpoint", C.c_int),
                ("weights", C.c_void_p), ("profile", C.c_void_p), ("efficiency", C.c_void_p)]


class HgcOsprCfg(C.Structure):
    _fields_ = [("variant", C.c_int), ("subframes", C.c_int), ("seed", C.c_uint64),
                ("feedback_gain", C.c_double), ("freedom_scale", C.c_int)]


class HgcOsprIo(C.Structure):
    _fields_ = [("amplitude", C.c_void_p), ("per_job_target", C.c_int), ("roi", C.c_void_p),
                ("seeds", C.c_void_p), ("levels8", C.c_void_p), ("levels16", C.c_void_p),
                ("frames", C.c_void_p), ("frame_mse", C.c_void_p), ("cumulative_mse", C.c_void_p),
                ("mean_intensity", C.c_void_p), ("replay", C.c_void_p), ("final_error", C.c_void_p),
                ("seconds", C.c_void_p), ("frames_gray8", C.c_void_p), ("replay_gray8", C.c_void_p),
                ("replay_peak", C.c_void_p), ("levels1", C.c_void_p), ("profile", C.c_void_p)]


class HgcIftaIo64(C.Structure):
    _fields_ = [("amplitude", C.c_void_p), ("phase", C.c_void_p), ("roi", C.c_void_p), ("init_field", C.c_void_p),
                ("init_weights", C.c_void_p), ("hologram", C.c_void_p), ("replay", C.c_void_p),
                ("levels", C.c_void_p), ("trace", C.c_void_p), ("final_error", C.c_void_p),
                ("fresnel_q", C.c_void_p), ("profile", C.c_void_p)]


class HgcOsprIo64(C.Structure):
    _fields_ = [("amplitude", C.c_void_p), ("roi", C.c_void_p), ("frames", C.c_void_p), ("levels", C.c_void_p),
                ("frame_mse", C.c_void_p), ("cumulative_mse", C.c_void_p), ("mean_intensity", C.c_void_p),
                ("replay", C.c_void_p), ("final_error", C.c_void_p), ("profile", C.c_void_p)]


_vp, _i, _u64, _d = C.c_void_p, C.c_int, C.c_uint64, C.c_double
_P = C.POINTER

_SIGS = {
    "hgc_abi_version": (_i, []),
    "hgc_last_error": (C.c_char_p, []),
    "hgc_device_count": (_i, [_P(_i)]),
    "hgc_set_device": (_i, [_i]),
    "hgc_max_side": (_i, []),
    "hgc_ifta_run": (_i, [_P(HgcIftaCfg), _P(HgcSlm), _P(HgcFresnel), _i, _i, _i, _P(HgcIftaIo)]),
    "hgc_ospr_run": (_i, [_P(HgcOsprCfg), _P(HgcSlm), _i, _i, _i, _P(HgcOsprIo)]),
    "hgc_ospr_run_fresnel": (_i, [_P(HgcOsprCfg), _P(HgcSlm), _P(HgcFresnel), _i, _i, _i, _P(HgcOsprIo)]),
    "hgc_ospr_plan_set_fresnel": (_i, [_vp, _P(HgcFresnel)]),
    "hgc_ifta_plan_create": (_i, [_P(_vp), _P(HgcIftaCfg), _P(HgcSlm), _P(HgcFresnel), _i, _i, _i]),
    "hgc_ifta_plan_upload": (_i, [_vp, _P(HgcIftaIo)]),
    "hgc_ifta_plan_execute": (_i, [_vp, _vp]),
    "hgc_ifta_plan_download": (_i, [_vp, _P(HgcIftaIo)]),
    "hgc_ifta_plan_device_ptrs": (_i, [_vp, _P(_vp), _P(_vp), _P(_vp)]),
    "hgc_ifta_plan_launches": (_i, [_vp]),
    "hgc_ifta_plan_profile": (_i, [_vp, _i, _P(_d), _P(_d), _P(_d)]),
    "hgc_ifta_plan_set_kernel_timing": (_i, [_vp, _i]),
    "hgc_ifta_plan_kernel_times": (_i, [_vp, _P(_d), _P(_d), _P(_i)]),
    "hgc_ifta_plan_destroy": (_i, [_vp]),
    "hgc_ospr_plan_create": (_i, [_P(_vp), _P(HgcOsprCfg), _P(HgcSlm), _i, _i, _i, _i]),
    "hgc_ospr_plan_upload": (_i, [_vp, _P(HgcOsprIo)]),
    "hgc_ospr_plan_execute": (_i, [_vp, _vp]),
    "hgc_ospr_plan_download": (_i, [_vp, _P(HgcOsprIo)]),
    "hgc_ospr_plan_device_ptrs": (_i, [_vp, _P(_vp), _P(_vp), _P(_vp)]),
    "hgc_ospr_plan_launches": (_i, [_vp]),
    "hgc_ospr_plan_profile": (_i, [_vp, _i, _P(_d), _P(_d), _P(_d), _P(_d)]),
    "hgc_ospr_block_plan_create": (_i, [_P(_vp), _P(HgcOsprCfg), _P(HgcSlm), _i, _i, _i, _i]),
    "hgc_ospr_block_sum": (_i, [_vp, _P(_vp), _P(C.c_size_t)]),
    "hgc_ospr_block_finish": (_i, [_vp, _vp, _i, _i, _vp]),
    "hgc_ospr_plan_destroy": (_i, [_vp]),
    "hgc_fft2d": (_i, [_i, _i, _i, _i, _vp, _vp]),
    "hgc_fft2d_f64": (_i, [_i, _i, _i, _i, _vp, _vp]),
    "hgc_propagate": (_i, [_i, _i, _i, _P(HgcFresnel), _i, _vp, _vp]),
    "hgc_quantise": (_i, [_P(HgcSlm), _i, _i, _i, _vp, _vp]),
    "hgc_seed_random_phase": (_i, [_vp, _i, _i, _u64, _u64, _vp]),
    "hgc_mt_jump_state": (_i, [_u64, _u64, _vp]),
    "hgc_batch_run": (_i, [_vp, _i, _i, C.c_size_t]),
    "hgc_ifta_run_f64": (_i, [_P(HgcIftaCfg), _P(HgcSlm), _P(HgcFresnel), _i, _i, _P(HgcIftaIo64)]),
    "hgc_ospr_run_f64": (_i, [_P(HgcOsprCfg), _P(HgcSlm), _i, _i, _P(HgcOsprIo64)]),
    "hgc_set_device_policy": (_i, [_i]),
    "hgc_write_field_dump": (_i, [C.c_char_p, _i, _i, _i, _vp]),
    "hgc_read_field_dump": (_i, [C.c_char_p, _P(_i), _P(_i), _P(_i), _vp]),
    "hgc_levels_to_gray8": (_i, [_vp, _i, _i, _i, _vp]),
    "hgc_gray8_to_levels": (_i, [_vp, C.c_size_t, _i, _vp]),
    "hgc_replay_to_gray8": (_i, [_vp, _i, _i, _i, _vp, _vp]),
    "hgc_write_replay_scale": (_i, [C.c_char_p, _d]),
    "hgc_write_png_gray": (_i, [C.c_char_p, _vp, _i, _i]),
    "hgc_smooth_blobs": (_i, [_i, _i, _vp]),
    "hgc_normalize_image": (_i, [_vp, C.c_size_t, _i]),
    "hgc_read_png_gray8": (_i, [C.c_char_p, _P(_i), _P(_i), _vp]),
    "hgc_fork_seed": (_u64, [_u64, _u64]),
    "hgc_mse": (_i, [_vp, _vp, _vp, _i, _i, _i, _P(_d)]),
    "hgc_fresnel_phase": (_i, [_i, _i, _P(HgcFresnel), _vp]),
    "hgc_subframe_mse_statistic": (_d, [_vp, _i]),
}

for _name, (_res, _args) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args

ABI_VERSION = 5  # HGC_ABI_VERSION of include/hologen_b200.h this binding was written against
if lib.hgc_abi_version() != ABI_VERSION:
    raise ImportError(f"{LIB_PATH}: ABI version {lib.hgc_abi_version()} != {ABI_VERSION}; rebuild the library")


def last_error() -> str:
    return lib.hgc_last_error().decode(errors="replace")


def check(rc: int) -> None:
    """Map an hgc_status to the reference's exception classes."""
    if rc == HGC_OK:
        return
    msg = last_error()
    if rc == HGC_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if rc == HGC_EUNSUPPORTED:
        raise HgcUnsupported(msg)
    if rc == HGC_EIO:
        raise HgcIOError(msg)
    raise HgcError(msg)


def exported_symbols() -> list[str]:
    return list(_SIGS)
