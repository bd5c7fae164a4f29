"""CPU: the output formats at the path's boundary, checked
against the reference's own io tests (proj/tests/test_io.cpp)."""
import os

import numpy as np
import pytest

import paper_2008_12214_b200 as hg
from paper_2008_12214_b200 import io as hio


def test_field_dump_round_trips_bit_for_bit(tmp_path):
    # test_io.cpp:103-133
    r = np.random.default_rng(5)
    f64 = (r.uniform(-3, 3, (5, 7)) + 1j * r.uniform(-3, 3, (5, 7))).astype(np.complex128)
    p64 = tmp_path / "field64.hgf"
    hio.write_field_dump(p64, f64)
    back = hio.read_field_dump(p64)
    assert back.dtype == np.complex128 and back.shape == (5, 7)
    assert np.array_equal(back.view(np.uint64), f64.view(np.uint64))
    f32 = (r.uniform(-3, 3, (4, 3)) + 1j * r.uniform(-3, 3, (4, 3))).astype(np.complex64)
    p32 = tmp_path / "field32.hgf"
    hio.write_field_dump(p32, f32)
    back32 = hio.read_field_dump(p32)
    assert back32.dtype == np.complex64 and np.array_equal(back32.view(np.uint32), f32.view(np.uint32))
    raw = p64.read_bytes()
    assert raw[:4] == b"HGF1" and raw[4] == 7 and raw[8] == 5 and raw[12] == 8
    assert len(raw) == 13 + 7 * 5 * 16
    # little-endian IEEE payload, row-major (re, im)
    assert np.array_equal(np.frombuffer(raw[13:], "<f8"), f64.view(np.float64).ravel())


def _hdr(nx, ny, code):
    return b"HGF1" + int(nx).to_bytes(4, "little") + int(ny).to_bytes(4, "little") + bytes([code])


@pytest.mark.parametrize("content,msg", [
    (b"NOPE" + bytes(9), "not an HGF1"),
    (_hdr(2, 2, 2), "16-bit fields are not enabled"),
    (_hdr(2, 2, 3), "unknown precision code"),
    (_hdr(2, 2, 4), "size mismatch"),
    (_hdr(0, 2, 4), "implausible dimensions"),
])
def test_field_dump_rejects_malformed_files(tmp_path, content, msg):
    # test_io.cpp:135-176: std::runtime_error with these messages
    p = tmp_path / "bad.hgf"
    p.write_bytes(content)
    with pytest.raises(hg.HgcIOError, match=msg):
        hio.read_field_dump(p)


def test_field_dump_missing_file_and_non_finite(tmp_path):
    with pytest.raises(hg.HgcIOError, match="cannot open"):
        hio.read_field_dump(tmp_path / "does_not_exist.hgf")
    f = np.zeros((2, 2), np.complex128)
    f[0, 1] = np.nan
    with pytest.raises(ValueError, match="non-finite"):  # test_io.cpp:178-183
        hio.write_field_dump(tmp_path / "nan.hgf", f)


def test_hologram_png_encoding_is_lossless_up_to_256_levels():
    # test_io.cpp:199-224
    r = np.random.default_rng(9)
    for levels in (2, 17, 256):
        idx = r.integers(0, levels, (4, 6)).astype(np.int32)
        idx[0, 0], idx[0, 1] = 0, levels - 1
        px = hio.levels_to_gray8(idx, levels)
        want = np.floor(255.0 * idx / (levels - 1) + 0.5).astype(np.uint8)  # lround, non-negative
        assert np.array_equal(px, want)
        assert np.array_equal(hio.gray8_to_levels(px, levels), idx)
    idx = np.zeros((2, 2), np.int32)
    with pytest.raises(ValueError, match=r"\[2, 256\]"):
        hio.levels_to_gray8(idx, 257)
    with pytest.raises(ValueError, match=r"\[2, 256\]"):
        hio.levels_to_gray8(idx, 1)
    idx[1, 0] = 5
    with pytest.raises(ValueError, match="out of range"):
        hio.levels_to_gray8(idx, 4)
    with pytest.raises(ValueError, match=r"\[2, 256\]"):
        hio.gray8_to_levels(np.zeros(4, np.uint8), 1)


def test_replay_scale_text(tmp_path):
    # test_io.cpp:327-342: "amplitude_at_255=4\n", "=0\n" (std::to_chars shortest form)
    p = tmp_path / "replay.png"
    hio.write_replay_scale(p, 4.0)
    assert open(str(p) + ".scale.txt").read() == "amplitude_at_255=4\n"
    hio.write_replay_scale(p, 0.0)
    assert open(str(p) + ".scale.txt").read() == "amplitude_at_255=0\n"
    hio.write_replay_scale(p, 0.1 + 0.2)
    assert open(str(p) + ".scale.txt").read() == "amplitude_at_255=0.30000000000000004\n"
