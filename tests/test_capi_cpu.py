"""CPU: the C ABI library loads and exports every symbol include/*.h
declares; host-side API logic (validation, value types) works without a
GPU; and compute calls fail loudly instead of falling back to the CPU."""
import re

import numpy as np
import pytest

import paper_2008_12214_b200 as hg
from paper_2008_12214_b200 import _lib
from conftest import has_gpu


def declared_symbols():
    txt = open(_lib.HEADER_PATH).read()
    decl = r"^(?:int|double|uint64_t|const char\*)\s+(hgc_\w+)\("
    return sorted(set(re.findall(decl, txt, re.M)))


def test_header_symbols_exported():
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(_lib.lib, s), s
    assert set(syms) <= set(_lib.exported_symbols()) | {"hgc_ifta_plan_profile", "hgc_ospr_plan_profile"}
    assert _lib.lib.hgc_abi_version() == _lib.ABI_VERSION == 5 and _lib.lib.hgc_max_side() == 4096


def test_fork_seed_matches_reference_rng():
    # Rng(seed).fork(0) engine seed, rng.hpp:42-44 (pinned against the oracle)
    from pyoracle import Oracle
    o = Oracle("restatement")
    for s in (0, 1, 12345, 2 ** 64 - 1):
        assert hg.fork_seed(s, 0) == o.fork_seed(s, 0)


def test_value_type_validation_messages():
    with pytest.raises(ValueError, match="levels must be >= 2"):
        hg.SlmSpec.phase(1, 0.0, 1.0)
    with pytest.raises(ValueError, match="full_circle requires a 2\\*pi range"):
        hg.SlmSpec(hg.SlmMode.Phase, 4, 0.0, 3.0, True).validate()
    with pytest.raises(ValueError, match="need 0 <= min_amp < max_amp"):
        hg.SlmSpec.amplitude(3, 1.0, 0.5)
    with pytest.raises(ValueError, match="wavelength must be positive"):
        hg.FresnelParams(0, 0.1, 8e-6, 8e-6).validate()
    t = hg.TargetSpec(np.ones((4, 4)))
    t.roi = np.zeros((4, 4), np.uint8)
    with pytest.raises(ValueError, match="roi covers no pixels"):
        t.validate()
    with pytest.raises(ValueError, match="iterations must be >= 1"):
        hg.IftaConfig(iterations=0, slm=hg.SlmSpec.binary_phase(), target=hg.TargetSpec(np.ones((4, 4)))).validate()
    with pytest.raises(ValueError, match="feedback_gain"):
        hg.OsprConfig(subframes=2, feedback_gain=2.0, slm=hg.SlmSpec.binary_phase(),
                      target=hg.TargetSpec(np.ones((4, 4)))).validate()
    assert hg.lt_area_fractions(10, 0.1)[-1] == 1.0 and abs(hg.lt_area_fractions(10, 0.1)[0] - 0.1) < 1e-12
    assert abs(hg.SlmSpec.amplitude(5).spacing() - 0.25) < 1e-15


def test_patterns_match_reference(ref_oracle):
    a = hg.patterns.smooth_blobs(48, 40)
    b = ref_oracle.smooth_blobs(48, 40)
    assert np.max(np.abs(a - b)) < 1e-15
    c = hg.normalize_image(a.copy(), hg.Normalization.UnitEnergy)
    d = ref_oracle.normalize(b)
    assert np.max(np.abs(c - d)) < 1e-13


def test_allowed_states_match_reference(ref_oracle):
    for spec in (hg.SlmSpec.binary_phase(), hg.SlmSpec.full_circle_phase(256), hg.SlmSpec.phase(17, -1.0, 1.0),
                 hg.SlmSpec.amplitude(7, 0.1, 1.3)):
        assert np.array_equal(hg.allowed_states_f32(spec), ref_oracle.quant_states(spec))


@pytest.mark.skipif(has_gpu(), reason="only meaningful without a GPU")
def test_no_cpu_fallback():
    with pytest.raises(hg.HgcError):
        hg.fft_forward(np.zeros((8, 8), np.complex64))
    with pytest.raises(hg.HgcError):
        hg.run_gs(hg.IftaConfig(iterations=1, slm=hg.SlmSpec.binary_phase(),
                                target=hg.TargetSpec(hg.patterns.bench_target(8))))


def _mt_next(window: np.ndarray, k: int) -> np.ndarray:
    """k tempered std::mt19937_64 outputs from a saved window (pos = 312)."""
    m = (1 << 64) - 1
    x = [int(v) for v in window]
    out = []
    for i in range(k):
        y = (x[i] & 0xFFFFFFFF80000000) | (x[i + 1] & 0x7FFFFFFF)
        w = x[i + 156] ^ (y >> 1) ^ (0xB5026F5AA96619E9 if y & 1 else 0)
        x.append(w)
        w ^= (w >> 29) & 0x5555555555555555
        w ^= (w << 17) & 0x71D67FFFEDA60000 & m
        w ^= (w << 37) & 0xFFF7EEE000000000 & m
        w ^= w >> 43
        out.append(w & m)
    return np.array(out, np.uint64)


@pytest.mark.parametrize("draws", [0, 1, 311, 312, 313, 4096 * 3 + 5, 1 << 24, 24 * (1 << 20) + 7])
def test_mt_jump_state_matches_sequential_stream(oracle, draws):
    """Jump-ahead (x^J mod the characteristic polynomial) lands exactly on draw J
    of the sequential engine (rng.hpp:23-34); the GPU seeds chunk k of a stream
    from these states."""
    es = hg.fork_seed(7, 0)
    w = hg.mt_jump_state(es, draws)
    nxt = _mt_next(w, 8)
    want = oracle.mt_draws(es, 8, skip=draws)
    np.testing.assert_array_equal(nxt, want)


def test_ospr_block_plan_validation():
    """Subframe-block plans reject adaptive OSPR (sequential:
    replicas only) and blocks outside the job before touching a device."""
    amp = hg.patterns.bench_target(32)
    base = dict(subframes=4, slm=hg.SlmSpec.binary_phase(), target=hg.TargetSpec(amp), seed=1)
    with pytest.raises(hg.HgcUnsupported, match="sequential"):
        hg.OsprBlockPlan(hg.OsprConfig(variant=hg.OsprVariant.AdaptiveOspr, **base), 32, 32, 0, 2)
    with pytest.raises(ValueError, match="outside"):
        hg.OsprBlockPlan(hg.OsprConfig(**base), 32, 32, 3, 2)
    with pytest.raises(ValueError, match="count"):
        hg.OsprBlockPlan(hg.OsprConfig(**base), 32, 32, 0, 0)


def test_bench_target_bit_identical_to_reference_generator(ref_oracle):
    # patterns::smooth_blobs + normalize_image(UnitEnergy) (patterns.hpp:55-80,
    # target.hpp:15-30), the reference bench's target (bench.cpp:115-116)
    for n in (16, 64, 1024):
        got = hg.patterns.bench_target(n)
        want = ref_oracle.normalize(ref_oracle.smooth_blobs(n, n), True)
        assert np.array_equal(got, want)
    assert np.array_equal(hg.patterns.smooth_blobs(40, 24), ref_oracle.smooth_blobs(40, 24))


def test_missing_library_fails_import(tmp_path):
    """No silent fallback when the sm_100a library is absent: importing the
    package raises (subprocess, so this session's loaded library is untouched)."""
    import subprocess
    import sys
    env = dict(__import__("os").environ, HG_LIB=str(tmp_path / "absent.so"))
    r = subprocess.run([sys.executable, "-c", "import paper_2008_12214_b200"], cwd=_lib._HERE + "/..", env=env,
                       capture_output=True, text=True)
    assert r.returncode != 0 and "ImportError" in r.stderr and "build the sm_100a library" in r.stderr
