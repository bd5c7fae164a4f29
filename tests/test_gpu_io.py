"""GPU: device-side output encodings — write_replay_png and
write_hologram_png pixels computed from the resident results."""
import ctypes
import ctypes.util

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
hg = pytest.importorskip("paper_2008_12214_b200")
hio = hg.io


_libm = ctypes.CDLL(ctypes.util.find_library("m"))
_libm.hypot.restype = ctypes.c_double
_libm.hypot.argtypes = [ctypes.c_double, ctypes.c_double]
_hypot = np.vectorize(_libm.hypot, otypes=[np.float64])


def _replay_px(replay):
    """io.cpp:189-205 on the host: amp = std::abs(complex<double>) = libm hypot
    (numpy's SIMD complex abs rounds differently), px = lround(amp * 255/peak)."""
    z = np.asarray(replay)
    amp = _hypot(z.real.astype(np.float64), z.imag.astype(np.float64))
    peak = amp.max()
    if peak == 0:
        return np.zeros(amp.shape, np.uint8), 0.0
    return np.clip(np.floor(amp * (255.0 / peak) + 0.5), 0, 255).astype(np.uint8), peak


def test_replay_png_known_answer():
    # test_io.cpp:327-342
    r = np.array([[0, 1j], [-2, -4j]], np.complex64)
    px, peak = hio.replay_to_gray8(r)
    assert px.ravel().tolist() == [0, 64, 128, 255] and peak == 4.0
    px, peak = hio.replay_to_gray8(np.zeros((2, 2), np.complex64))
    assert px.ravel().tolist() == [0, 0, 0, 0] and peak == 0.0


def test_replay_png_matches_host_encoding():
    r = np.random.default_rng(2)
    z = (r.normal(size=(96, 80)) + 1j * r.normal(size=(96, 80))).astype(np.complex64)
    px, peak = hio.replay_to_gray8(z)
    want, wpeak = _replay_px(z)
    assert peak == wpeak
    assert np.array_equal(px, want)


def test_ifta_plan_gray_outputs():
    amp = hg.patterns.bench_target(128)
    cfg = hg.IftaConfig(iterations=4, slm=hg.SlmSpec.full_circle_phase(16), target=hg.TargetSpec(amp), seed=1)
    p = hg.IftaPlan(cfg, 128, 128, 2)
    p.upload(np.broadcast_to(amp, (2, 128, 128)), seeds=[1, 2])
    p.execute()
    out = p.download(gray=True)
    for b in range(2):
        assert np.array_equal(out.hologram_gray8[b], hio.levels_to_gray8(out.levels[b].astype(np.int32), 16))
        want, peak = _replay_px(out.replay[b])
        assert out.replay_peak[b] == peak
        assert np.array_equal(out.replay_gray8[b], want)


def test_ospr_plan_gray_outputs():
    amp = hg.patterns.bench_target(64)
    cfg = hg.OsprConfig(subframes=3, slm=hg.SlmSpec.binary_phase(), target=hg.TargetSpec(amp), seed=4)
    p = hg.OsprPlan(cfg, 64, 64, 2)
    p.upload(amp, seeds=[4, 5])
    p.execute()
    out = p.download(gray=True)
    for j in range(2):
        for n in range(3):
            assert np.array_equal(out["frames_gray8"][j, n], hio.levels_to_gray8(out["levels"][j, n].astype(np.int32), 2))
        replay = np.sqrt(out["mean_intensity"][j]).astype(np.float32).astype(np.complex64)  # ospr.hpp:152-156
        want, peak = _replay_px(replay)
        assert out["replay_peak"][j] == peak
        assert np.array_equal(out["replay_gray8"][j], want)


def test_ospr_binary_bitplanes():
    """2-level SLM frames as bit-planes (hgc_ospr_io.levels1): np.packbits(little) of the levels."""
    amp = hg.patterns.bench_target(64)
    cfg = hg.OsprConfig(subframes=3, slm=hg.SlmSpec.binary_phase(), target=hg.TargetSpec(amp), seed=2)
    p = hg.OsprPlan(cfg, 64, 64, 2)
    p.upload(amp, seeds=[2, 3])
    p.execute()
    out = p.download(bits=True)
    want = np.packbits(out["levels"].reshape(2, 3, -1), axis=-1, bitorder="little")
    assert np.array_equal(out["levels1"], want)
    p16 = hg.OsprPlan(hg.OsprConfig(subframes=1, slm=hg.SlmSpec.full_circle_phase(4), target=hg.TargetSpec(amp)),
                      64, 64, 1)
    p16.upload(amp)
    p16.execute()
    with pytest.raises(ValueError, match="2-level"):
        p16.download(bits=True)
