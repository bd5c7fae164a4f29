"""Synthetic targets, patterns.hpp:10-83 (input generators for tests and the
benchmark; the reference's own benchmark target is smooth_blobs + UnitEnergy,
bench.cpp:115-116)."""
from __future__ import annotations

import numpy as np

from .types import Normalization, normalize_image


def checkerboard(width: int, height: int, cell: int = 8) -> np.ndarray:  # patterns.hpp:14-21
    if cell < 1:
        raise ValueError("checkerboard: cell must be >= 1")
    y, x = np.mgrid[0:height, 0:width]
    return (((x // cell + y // cell) & 1) != 0).astype(np.float64)


def letter_a(width: int, height: int) -> np.ndarray:  # patterns.hpp:25-36
    rows = [0x18, 0x3C, 0x66, 0x66, 0x7E, 0x66, 0x66, 0x00]
    y, x = np.mgrid[0:height, 0:width]
    by = (y.astype(np.int64) * 8) // height
    bx = (x.astype(np.int64) * 8) // width
    r = np.array(rows, dtype=np.int64)[by]
    return ((r >> (7 - bx)) & 1).astype(np.float64)


def spot_array(width: int, height: int, spots_x: int = 4, spots_y: int = 4) -> np.ndarray:  # patterns.hpp:39-51
    if spots_x < 1 or spots_y < 1 or spots_x > width or spots_y > height:
        raise ValueError("spot_array: spot counts must fit the image")
    img = np.zeros((height, width))
    for j in range(spots_y):
        yy = int((j + 0.5) * height / spots_y)
        for i in range(spots_x):
            img[yy, int((i + 0.5) * width / spots_x)] = 1.0
    return img


_BLOBS = ((0.30, 0.35, 0.16, 1.00), (0.68, 0.28, 0.10, 0.75), (0.62, 0.70, 0.20, 0.90), (0.22, 0.74, 0.08, 0.60))


def smooth_blobs(width: int, height: int) -> np.ndarray:  # patterns.hpp:55-80
    """Bit-identical to the reference's (hgc_smooth_blobs: same operation
    order and the C library's exp; numpy's vectorised exp differs in the last
    bit on some inputs)."""
    from ._lib import check, lib
    if width < 1 or height < 1:
        raise ValueError("RealImage: dimensions must be positive")
    img = np.empty((height, width), np.float64)
    check(lib.hgc_smooth_blobs(width, height, img.ctypes.data))
    return img


def bench_target(n: int) -> np.ndarray:
    """smooth_blobs + UnitEnergy, the reference's benchmark target (bench.cpp:115-116)."""
    return normalize_image(smooth_blobs(n, n), Normalization.UnitEnergy)
