"""GPU parity of the primitive operators against the CPU oracle.

Reference anchors: FFT contract fft.hpp:17-27 + fixtures test_fft.cpp:28-51;
quantiser quantise.hpp:175-216 (bit-exact levels); seed_random_phase
rng.hpp:54-67 (bit-exact field); make_fresnel_phase propagation.hpp:36-54;
mse metrics.hpp:70-124.
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

hg = pytest.importorskip("paper_2008_12214_b200")
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rand_field(shape, seed, scale=1.0):
    r = np.random.default_rng(seed)
    return (r.uniform(-scale, scale, shape) + 1j * r.uniform(-scale, scale, shape)).astype(np.complex64)


def test_fft_4x4_golden():
    g = json.load(open(os.path.join(GOLDEN, "fft_4x4.json")))
    x = (np.array(g["in_re"]) + 1j * np.array(g["in_im"])).reshape(4, 4).astype(np.complex64)
    want = (np.array(g["out_re"]) + 1j * np.array(g["out_im"])).reshape(4, 4)
    got = hg.fft_forward(x)
    assert np.max(np.abs(got - want)) < 2e-6  # f32 transform of the f64 fixture (test_fft.cpp:75-88 at 1e-12 in f64)


@pytest.mark.parametrize("n", [2, 4, 8, 16, 64, 256, 512, 1024, 2048, 4096])
def test_fft_matches_oracle(oracle, n):
    ny = n
    nx = n if n != 64 else 128  # one rectangular case
    x = rand_field((ny, nx), 100 + n)
    for sign in (-1, +1):
        got = hg.fft_forward(x) if sign < 0 else hg.fft_inverse(x)
        if n <= 1024:
            ref = oracle.fft2(x.astype(np.complex128), sign)
        else:  # numpy double FFT as the exact reference at large sizes
            f = np.fft.fft2(x.astype(np.complex128)) if sign < 0 else np.fft.ifft2(x.astype(np.complex128)) * x.size
            ref = f / np.sqrt(x.size)
        err = np.max(np.abs(got - ref))
        assert err < 2e-6 * np.sqrt(np.log2(x.size) + 1), (n, sign, err)


def test_fft_4x4_golden_f64():
    """fft_forward<double> on the GPU against the reference's 4x4 fixture at its own 1e-12 (test_fft.cpp:75-88)."""
    g = json.load(open(os.path.join(GOLDEN, "fft_4x4.json")))
    x = (np.array(g["in_re"]) + 1j * np.array(g["in_im"])).reshape(4, 4)
    want = (np.array(g["out_re"]) + 1j * np.array(g["out_im"])).reshape(4, 4)
    assert np.max(np.abs(hg.fft_forward(x) - want)) < 1e-12


@pytest.mark.parametrize("ny,nx", [(2, 2), (8, 16), (16, 2), (64, 128), (1024, 1024), (4096, 256), (256, 4096),
                                   (4096, 4096)])
def test_fft_f64_matches_numpy(ny, nx):
    r = np.random.default_rng(ny * 7 + nx)
    x = r.standard_normal((ny, nx)) + 1j * r.standard_normal((ny, nx))
    F = hg.fft_forward(x)
    assert F.dtype == np.complex128
    assert np.max(np.abs(F - np.fft.fft2(x) / np.sqrt(x.size))) < 1e-12 * np.sqrt(np.log2(x.size) + 1) * 4
    B = hg.fft_inverse(x)
    assert np.max(np.abs(B - np.fft.ifft2(x) * np.sqrt(x.size))) < 1e-12 * np.sqrt(np.log2(x.size) + 1) * 4
    if ny * nx <= 1 << 20:  # batched, via the C ABI directly
        from paper_2008_12214_b200 import _lib
        xb = np.stack([x, 2 * x])
        out = np.empty_like(xb)
        _lib.check(_lib.lib.hgc_fft2d_f64(nx, ny, -1, 2, xb.ctypes.data, out.ctypes.data))
        assert np.array_equal(out[0], F) and np.max(np.abs(out[1] - 2 * F)) < 1e-11


def test_fft_delta_constant_roundtrip():
    f = np.zeros((8, 8), np.complex64)
    f[0, 0] = 1
    F = hg.fft_forward(f)
    assert np.allclose(F, 1 / 8, atol=1e-7)
    c = np.full((16, 16), 0.5 - 0.25j, np.complex64)
    C = hg.fft_forward(c)
    assert abs(C[0, 0] - (8 - 4j)) < 1e-5 and np.max(np.abs(C.ravel()[1:])) < 1e-5
    x = rand_field((256, 256), 7)
    back = hg.fft_inverse(hg.fft_forward(x))
    assert np.max(np.abs(back - x)) < 1e-5
    e_in, e_out = np.sum(np.abs(x.astype(np.complex128)) ** 2), np.sum(np.abs(hg.fft_forward(x).astype(np.complex128)) ** 2)
    assert abs(e_out - e_in) / e_in < 1e-6


def test_fft_rejects_unsupported_and_nonfinite():
    with pytest.raises(hg.HgcUnsupported):  # non-powers of two are covered up to 2048 per side
        hg.fft_forward(np.zeros((5, 3000), np.complex64))
    bad = np.zeros((8, 8), np.complex64)
    bad[1, 1] = np.nan
    with pytest.raises(ValueError):
        hg.fft_forward(bad)
    bad7 = np.zeros((5, 7), np.complex64)
    bad7[2, 3] = np.inf
    with pytest.raises(ValueError, match="non-finite"):
        hg.fft_forward(bad7)


@pytest.mark.parametrize("ny,nx", [(5, 7), (16, 3), (1, 1), (3, 1), (1, 5), (12, 64), (100, 30), (1080, 1920)])
def test_fft_any_size_matches_numpy(ny, nx):
    """FftBackend accepts any nx, ny >= 1 (fft.hpp:17-27; test_fft.cpp:90-98 uses 5x7 and 16x3):
    non-powers of two go through Bluestein in double, for both precisions."""
    r = np.random.default_rng(ny * 31 + nx)
    x = r.standard_normal((ny, nx)) + 1j * r.standard_normal((ny, nx))
    ref_f = np.fft.fft2(x) / np.sqrt(x.size)
    ref_i = np.fft.ifft2(x) * np.sqrt(x.size)
    tol = 1e-12 * np.sqrt(np.log2(x.size) + 2) * 8
    assert np.max(np.abs(hg.fft_forward(x) - ref_f)) < tol
    assert np.max(np.abs(hg.fft_inverse(x) - ref_i)) < tol
    x32 = x.astype(np.complex64)
    ref32 = np.fft.fft2(x32.astype(np.complex128)) / np.sqrt(x.size)
    got32 = hg.fft_forward(x32)
    assert got32.dtype == np.complex64
    assert np.max(np.abs(got32 - ref32)) < 2e-6 * np.sqrt(np.log2(x.size) + 2)  # double inside, one float rounding


SLMS = {
    "binary": lambda: hg.SlmSpec.binary_phase(),
    "fc4": lambda: hg.SlmSpec.full_circle_phase(4),
    "fc5": lambda: hg.SlmSpec.full_circle_phase(5),
    "fc256": lambda: hg.SlmSpec.full_circle_phase(256),
    "fc256_offset": lambda: hg.SlmSpec.full_circle_phase(256, 0.3),
    "r17": lambda: hg.SlmSpec.phase(17, -hg.PI / 2, hg.PI / 2),
    "r3": lambda: hg.SlmSpec.phase(3, 0.4, 1.1),
    "r2q": lambda: hg.SlmSpec.phase(2, 0.0, hg.PI / 2),
    "amp2": lambda: hg.SlmSpec.binary_amplitude(),
    "amp7": lambda: hg.SlmSpec.amplitude(7, 0.1, 1.3),
    "amp9": lambda: hg.SlmSpec.amplitude(9, 0.25, 0.75),
}


@pytest.mark.parametrize("name", list(SLMS))
def test_quantiser_bit_exact(oracle, name):
    spec = SLMS[name]()
    f = rand_field((256, 256), 552, 2.0)
    # edge cases: exact zeros, exact axes, exact level angles, ties
    f[0, :8] = [0, 1, -1, 1j, -1j, 1 + 1j, -1 - 1j, 0.5]
    got = f.copy()
    lv = hg.Quantiser(spec, 256, 256).apply(got, levels_out=True)
    ref_f, ref_lv = oracle.quantise(spec, f)
    assert np.array_equal(lv, ref_lv)
    assert np.array_equal(got.view(np.uint32), ref_f.view(np.uint32))


@pytest.mark.parametrize("mode", ["phase", "amplitude"])
def test_quantiser_illumination_bit_exact(oracle, mode):
    r = np.random.default_rng(600)
    il = r.uniform(0.5, 2.0, (50, 64)) * np.exp(1j * r.uniform(0, hg.TWO_PI, (50, 64)))
    spec = hg.SlmSpec.full_circle_phase(4) if mode == "phase" else hg.SlmSpec.amplitude(7, 0.1, 1.3)
    spec.illumination = il
    f = rand_field((50, 64), 552, 2.0)
    got = f.copy()
    lv = hg.Quantiser(spec, 64, 50).apply(got, levels_out=True)
    ref_f, ref_lv = oracle.quantise(spec, f)
    assert np.array_equal(lv, ref_lv)
    assert np.array_equal(got.view(np.uint32), ref_f.view(np.uint32))


def test_quantiser_tie_goes_to_pi_state(oracle):
    # all-i field against {1, -1}: tie at half spacing rounds to the pi state (test_quantise.cpp:227-232)
    f = np.full((4, 4), 1j, np.complex64)
    lv = hg.Quantiser(hg.SlmSpec.binary_phase(), 4, 4).apply(f, levels_out=True)
    assert np.all(lv == 1)


@pytest.mark.parametrize("n,skip", [(64, 0), (512, 0), (300, 5), (1024, 3 * 1024 * 1024 + 17)])
def test_seed_random_phase_bit_exact(oracle, n, skip):
    amp = hg.patterns.bench_target(n) if n != 300 else np.random.default_rng(1).uniform(0, 2, (n, 257))
    amp[0, :3] = 0.0  # zero-amplitude pixels still consume a draw (rng.hpp:51-53)
    got = hg.seed_random_phase(amp, seed=7, skip=skip)
    ref = oracle.seed_random_phase(amp, 7, skip=skip)  # Rng(7).fork(0) inside
    mism = np.count_nonzero(got.view(np.uint32) != ref.view(np.uint32))
    assert mism <= 1, mism  # CUDA vs glibc double sincos may differ by 1 ulp (~2^-29 per value)


@pytest.mark.parametrize("chunks,skip", [(2, 0), (3, 0), (7, 1000), (64, 0), (5, 3 * 512 * 512 + 1)])
def test_seed_chunked_jump_ahead_bit_exact(oracle, monkeypatch, chunks, skip):
    """One stream split across CTAs by MT jump-ahead (k_mt_jump) must equal the
    sequential stream: chunk boundaries at draw offsets that are not multiples
    of the 312-word twist block, with and without a skip."""
    monkeypatch.setenv("HG_SEED_CHUNKS", str(chunks))
    amp = np.random.default_rng(3).uniform(0, 2, (512, 512))
    got = hg.seed_random_phase(amp, seed=11, skip=skip)
    ref = oracle.seed_random_phase(amp, 11, skip=skip)
    mism = np.count_nonzero(got.view(np.uint32) != ref.view(np.uint32))
    assert mism <= 1, mism


def test_seed_default_chunking_full_size(oracle):
    """4096^2 (16.7M draws) with the default chunking (~2 CTAs per SM)."""
    amp = hg.patterns.bench_target(4096)
    got = hg.seed_random_phase(amp, seed=5)
    ref = oracle.seed_random_phase(amp, 5)
    mism = np.count_nonzero(got.view(np.uint32) != ref.view(np.uint32))
    assert mism <= 4, mism


def test_fresnel_phase_matches(oracle):
    p = hg.FresnelParams(532e-9, 0.1, 8e-6, 8e-6)
    got = hg.make_fresnel_phase(512, 256, p)
    ref = oracle.fresnel_q(512, 256, 532e-9, 0.1, 8e-6, 8e-6)
    mism = np.count_nonzero(got.view(np.uint32) != ref.view(np.uint32))
    assert mism <= 4, mism
    q8 = hg.make_fresnel_phase(8, 8, p)
    assert q8[4, 4] == 1 + 0j  # centre (test_propagation.cpp:62-68)


@pytest.mark.parametrize("scale_free", [False, True])
@pytest.mark.parametrize("masked", [False, True])
def test_mse_matches(oracle, scale_free, masked):
    t = hg.patterns.bench_target(128)
    r = rand_field((128, 128), 3)
    m = None
    if masked:
        m = np.zeros((128, 128), np.uint8)
        m[10:100, 20:90] = 1
    got = hg.mse(t, r, hg.MetricConfig(mask=m, scale_free=scale_free))
    ref = oracle.mse(t, r, m, scale_free)
    assert abs(got - ref) / ref < 1e-12


def test_mse_fixtures():
    # test_metrics.cpp:39-61, :130-149 (derive_fixtures.py)
    t = np.array([[1.0, 0.0]])
    r = np.array([[0.5, 0.5]], np.complex64)
    assert abs(hg.mse(t, r) - 0.25) < 1e-15
    assert abs(hg.mse(t, r, hg.MetricConfig(scale_free=True)) - 0.25) < 1e-12
    t4 = np.zeros((4, 4)); t4[:, :2] = 1
    r4 = np.zeros((4, 4), np.complex64); r4[:, :2] = 0.5
    m = np.zeros((4, 4), np.uint8); m[:, :2] = 1
    assert abs(hg.mse(t4, r4) - 0.125) < 1e-15
    assert abs(hg.mse(t4, r4, hg.MetricConfig(mask=m)) - 0.25) < 1e-15
