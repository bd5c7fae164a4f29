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


def _parse_png(data: bytes):
    """Independent PNG check: signature, CRCs, IHDR, and the inflated scanlines."""
    import struct
    import zlib
    assert data[:8] == b"\x89PNG\r\n\x1a\n"
    at, idat, ihdr = 8, b"", None
    while at < len(data):
        n, = struct.unpack(">I", data[at:at + 4])
        typ, body = data[at + 4:at + 8], data[at + 8:at + 8 + n]
        crc, = struct.unpack(">I", data[at + 8 + n:at + 12 + n])
        assert zlib.crc32(typ + body) == crc
        if typ == b"IHDR":
            ihdr = struct.unpack(">IIBBBBB", body)
        elif typ == b"IDAT":
            idat += body
        at += 12 + n
    w, h, depth, ctype, _, _, interlace = ihdr
    assert (depth, ctype, interlace) == (8, 0, 0)
    raw = zlib.decompress(idat)
    rows = [raw[y * (w + 1):(y + 1) * (w + 1)] for y in range(h)]
    assert all(r[0] == 0 for r in rows)  # filter type 0
    return np.frombuffer(b"".join(r[1:] for r in rows), np.uint8).reshape(h, w)


def test_hologram_png_round_trip(tmp_path):
    # write_hologram_png / read_hologram_png (io.cpp:272-298) as real PNG files
    from paper_2008_12214_b200 import io
    rng = np.random.default_rng(3)
    for L in (2, 7, 256):
        lv = rng.integers(0, L, size=(37, 53), dtype=np.int32)
        p = tmp_path / f"h{L}.png"
        io.write_hologram_png(p, lv, L)
        px = _parse_png(p.read_bytes())
        assert np.array_equal(px, io.levels_to_gray8(lv, L))
        assert np.array_equal(io.read_hologram_png(p, L), lv)
    with pytest.raises(ValueError, match="level count must be in"):
        io.write_hologram_png(tmp_path / "x.png", np.zeros((2, 2), np.int32), 300)


def test_png_reader_filters_and_errors(tmp_path):
    # read_png_gray8 accepts every scanline filter (what libpng would write)
    import struct
    import zlib
    from paper_2008_12214_b200 import io
    from paper_2008_12214_b200._lib import HgcIOError
    rng = np.random.default_rng(4)
    img = rng.integers(0, 256, size=(6, 9), dtype=np.uint8)
    w, h = 9, 6
    raw = b""
    prev = np.zeros(w, np.int64)
    for y in range(h):
        f = y % 5
        cur = img[y].astype(np.int64)
        out = []
        for x in range(w):
            a = cur[x - 1] if x else 0
            b = prev[x]
            c = prev[x - 1] if x else 0
            pred = [0, a, b, (a + b) // 2, None][f]
            if f == 4:
                p = a + b - c
                pa, pb, pc = abs(p - a), abs(p - b), abs(p - c)
                pred = a if (pa <= pb and pa <= pc) else (b if pb <= pc else c)
            out.append((cur[x] - pred) & 255)
        raw += bytes([f]) + bytes(out)
        prev = cur

    def chunk(t, b):
        return struct.pack(">I", len(b)) + t + b + struct.pack(">I", zlib.crc32(t + b))
    data = b"\x89PNG\r\n\x1a\n" + chunk(b"IHDR", struct.pack(">IIBBBBB", w, h, 8, 0, 0, 0, 0)) + \
        chunk(b"IDAT", zlib.compress(raw)) + chunk(b"IEND", b"")
    p = tmp_path / "f.png"
    p.write_bytes(data)
    assert np.array_equal(io.read_png_gray8(p), img)
    (tmp_path / "bad.png").write_bytes(b"not a png")
    with pytest.raises(HgcIOError, match="not a PNG file"):
        io.read_png_gray8(tmp_path / "bad.png")
