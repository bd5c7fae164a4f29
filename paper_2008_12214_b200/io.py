"""Output formats on either side of the hot path, mirroring
the reference's io.hpp: HGF1 field dumps (io.cpp:168-186, :316-345), the
hologram-PNG level encoding (io.cpp:272-298) and the replay-PNG pixels and
scale file (io.cpp:189-207), and the PNG files themselves (write_png_gray /
read_png_gray8, io.cpp:221-258: 8-bit greyscale, zlib deflate)."""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import _lib
from ._lib import check, lib


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def write_field_dump(path: str | os.PathLike, field: np.ndarray) -> None:
    """write_field_dump: complex64 -> precision code 4, complex128 -> 8."""
    f = np.asarray(field)
    if f.ndim != 2 or not np.iscomplexobj(f):
        raise ValueError("field dump: expected a 2-D complex field")
    code = 8 if f.dtype == np.complex128 else 4
    f = np.ascontiguousarray(f, np.complex128 if code == 8 else np.complex64)
    check(lib.hgc_write_field_dump(os.fsencode(path), f.shape[1], f.shape[0], code, _p(f)))


def read_field_dump(path: str | os.PathLike) -> np.ndarray:
    """read_field_dump: complex64 (code 4) or complex128 (code 8) [ny][nx]."""
    nx, ny, code = C.c_int(), C.c_int(), C.c_int()
    bp = os.fsencode(path)
    check(lib.hgc_read_field_dump(bp, C.byref(nx), C.byref(ny), C.byref(code), None))
    out = np.empty((ny.value, nx.value), np.complex64 if code.value == 4 else np.complex128)
    check(lib.hgc_read_field_dump(bp, C.byref(nx), C.byref(ny), C.byref(code), _p(out)))
    return out


def levels_to_gray8(levels: np.ndarray, level_count: int) -> np.ndarray:
    """write_hologram_png's pixels: lround(255 k / (L-1))."""
    lv = np.ascontiguousarray(levels, np.int32)
    if lv.ndim != 2:
        raise ValueError("write_hologram_png: level buffer does not match dimensions")
    out = np.empty(lv.shape, np.uint8)
    check(lib.hgc_levels_to_gray8(_p(lv), lv.shape[1], lv.shape[0], level_count, _p(out)))
    return out


def gray8_to_levels(px: np.ndarray, level_count: int) -> np.ndarray:
    """read_hologram_png's decoding: lround(px (L-1) / 255)."""
    g = np.ascontiguousarray(px, np.uint8)
    out = np.empty(g.shape, np.int32)
    check(lib.hgc_gray8_to_levels(_p(g), g.size, level_count, _p(out)))
    return out


def replay_to_gray8(replay: np.ndarray) -> tuple[np.ndarray, float]:
    """write_replay_png's pixels and amplitude_at_255 (computed on the GPU)."""
    r = np.ascontiguousarray(replay, np.complex64)
    if r.ndim != 2:
        raise ValueError("replay image: expected a 2-D complex field")
    out = np.empty(r.shape, np.uint8)
    peak = C.c_double()
    check(lib.hgc_replay_to_gray8(_p(r), r.shape[1], r.shape[0], 1, _p(out), C.byref(peak)))
    return out, peak.value


def write_replay_scale(png_path: str | os.PathLike, peak: float) -> None:
    """The '<png>.scale.txt' companion: 'amplitude_at_255=<shortest double>'."""
    check(lib.hgc_write_replay_scale(os.fsencode(png_path), float(peak)))


def write_png_gray(path: str | os.PathLike, pixels: np.ndarray) -> None:
    """write_png_gray (io.cpp:221-237): 8-bit greyscale PNG of [height][width] pixels."""
    px = np.ascontiguousarray(pixels, np.uint8)
    if px.ndim != 2:
        raise ValueError("write_png_gray: pixel buffer does not match dimensions")
    check(lib.hgc_write_png_gray(os.fsencode(path), _p(px), px.shape[1], px.shape[0]))


def read_png_gray8(path: str | os.PathLike) -> np.ndarray:
    """read_png_gray8 (io.cpp:239-258) for 8-bit greyscale PNGs."""
    w, h = C.c_int(), C.c_int()
    bp = os.fsencode(path)
    check(lib.hgc_read_png_gray8(bp, C.byref(w), C.byref(h), None))
    out = np.empty((h.value, w.value), np.uint8)
    check(lib.hgc_read_png_gray8(bp, C.byref(w), C.byref(h), _p(out)))
    return out


def write_hologram_png(path: str | os.PathLike, levels: np.ndarray, level_count: int) -> None:
    """write_hologram_png (io.cpp:272-287): levels as lround(255 k / (L-1)) grey."""
    if level_count < 2 or level_count > 256:
        raise ValueError("write_hologram_png: level count must be in [2, 256] for a lossless 8-bit encoding")
    write_png_gray(path, levels_to_gray8(levels, level_count))


def read_hologram_png(path: str | os.PathLike, level_count: int) -> np.ndarray:
    """read_hologram_png (io.cpp:289-298): the level indices back (int32)."""
    return gray8_to_levels(read_png_gray8(path), level_count)


def write_replay_png(path: str | os.PathLike, replay: np.ndarray) -> float:
    """write_replay_png (io.cpp:189-207): |replay| scaled to 255 at its peak, plus
    '<path>.scale.txt'.  Returns amplitude_at_255."""
    px, peak = replay_to_gray8(replay)
    write_png_gray(path, px)
    write_replay_scale(path, peak)
    return peak
