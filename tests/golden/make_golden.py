"""Regenerate the golden fixtures in tests/golden/ (run in the build
container, where /root/reference exists).

Sources:
* fft_4x4.json — the reference's own fixture: numpy default_rng(20260818)
  4x4 complex field and its unitary DFT, exactly as
  proj/tests/oracles/derive_fixtures.py:74-92 derives it; cross-checked
  against the literals pinned in proj/tests/test_fft.cpp:28-51.
* mt19937_64.json — the C++ standard's known answer ([rand.predef]: the
  10000th output of a default-constructed std::mt19937_64 is
  9981545732273789042) plus the first draws of Rng(seed).fork(0) streams
  produced by the reference's rng.hpp compiled here (oracle/_ref).
* ref_runs.npz — small GS / WGS / Fresnel-GS / OSPR / adaptive-OSPR runs and
  quantiser decisions produced by the reference ITSELF (its unmodified headers
  compiled into oracle/_ref/libhgref.so with the substitute FFT).
"""
import json
import os
import re
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from pyoracle import Oracle  # noqa: E402

PI = 3.1415926535897932384626433832795


class Slm:
    def __init__(self, mode, levels, min_arg=0.0, max_arg=0.0, full_circle=False, min_amp=0.0, max_amp=1.0,
                 illumination=None):
        self.mode, self.levels, self.min_arg, self.max_arg = mode, levels, min_arg, max_arg
        self.full_circle, self.min_amp, self.max_amp, self.illumination = full_circle, min_amp, max_amp, illumination


BINARY = Slm(1, 2, 0.0, PI)
FC256 = Slm(1, 256, 0.0, 2 * PI, True)


def fft_fixture():
    rng = np.random.default_rng(20260818)
    a = rng.standard_normal((4, 4)) + 1j * rng.standard_normal((4, 4))
    f = np.fft.fft2(a) / np.sqrt(a.size)
    src = "/root/reference/proj/tests/test_fft.cpp"
    if os.path.exists(src):
        txt = open(src).read()
        lit = {}
        for name in ("kIn4Re", "kIn4Im", "kOut4Re", "kOut4Im"):
            body = re.search(name + r"\[16\] = \{(.*?)\};", txt, re.S).group(1)
            lit[name] = np.array([float(v) for v in body.replace("\n", " ").split(",") if v.strip()])
        assert np.array_equal(lit["kIn4Re"], a.real.ravel()) and np.array_equal(lit["kIn4Im"], a.imag.ravel())
        assert np.allclose(lit["kOut4Re"], f.real.ravel(), rtol=0, atol=1e-15)
        assert np.allclose(lit["kOut4Im"], f.imag.ravel(), rtol=0, atol=1e-15)
    return {"source": "derive_fixtures.py:74-92 / test_fft.cpp:28-51", "in_re": a.real.ravel().tolist(),
            "in_im": a.imag.ravel().tolist(), "out_re": f.real.ravel().tolist(), "out_im": f.imag.ravel().tolist()}


def main():
    ref = Oracle("reference")
    json.dump(fft_fixture(), open(os.path.join(HERE, "fft_4x4.json"), "w"), indent=1)

    mt = {"kat_seed": 5489, "kat_index": 10000, "kat_value": 9981545732273789042,
          "kat_from_reference": int(ref.mt_draws(5489, 1, skip=9999)[0])}
    assert mt["kat_from_reference"] == mt["kat_value"]
    for seed in (0, 1, 42):
        es = ref.fork_seed(seed, 0)
        mt[f"fork0_seed{seed}"] = str(es)
        mt[f"draws_seed{seed}"] = [str(int(v)) for v in ref.mt_draws(es, 8)]
        mt[f"draws_seed{seed}_skip1000"] = [str(int(v)) for v in ref.mt_draws(es, 4, skip=1000)]
    json.dump(mt, open(os.path.join(HERE, "mt19937_64.json"), "w"), indent=1)

    out = {}
    amp32 = ref.normalize(ref.smooth_blobs(32, 32))
    amp64 = ref.normalize(ref.smooth_blobs(64, 64))
    out["amp32"], out["amp64"] = amp32, amp64
    r = ref.ifta(amp64, BINARY, 20, seed=1)
    out["gs64_bin_levels"], out["gs64_bin_trace"], out["gs64_bin_replay"] = r.levels.astype(np.uint8), r.trace, r.replay
    r = ref.ifta(amp64, FC256, 10, seed=3)
    out["gs64_256_levels"], out["gs64_256_trace"] = r.levels.astype(np.uint8), r.trace
    r = ref.ifta(amp64, FC256, 10, seed=3, variant="wgs")
    out["wgs64_256_levels"], out["wgs64_256_trace"] = r.levels.astype(np.uint8), r.trace
    r = ref.ifta(amp32, FC256, 8, seed=9, fresnel=(532e-9, 0.1, 8e-6, 8e-6))
    out["fresnel32_levels"], out["fresnel32_trace"] = r.levels.astype(np.uint8), r.trace
    o = ref.ospr(amp32, BINARY, 6, seed=42)
    out["ospr32_levels"], out["ospr32_frame_mse"], out["ospr32_cum_mse"] = o.levels.astype(np.uint8), o.frame_mse, \
        o.cumulative_mse
    out["ospr32_mean_intensity"] = o.mean_intensity
    o = ref.ospr(amp32, BINARY, 4, seed=43, adaptive=True, gain=1.0)
    out["aospr32_levels"], out["aospr32_cum_mse"] = o.levels.astype(np.uint8), o.cumulative_mse
    rng = np.random.default_rng(552)
    f = (rng.uniform(-2, 2, (40, 40)) + 1j * rng.uniform(-2, 2, (40, 40))).astype(np.complex64)
    out["quant_in"] = f
    for name, spec in {"binary": BINARY, "fc256": FC256, "r17": Slm(1, 17, -PI / 2, PI / 2),
                       "amp7": Slm(0, 7, min_amp=0.1, max_amp=1.3)}.items():
        qf, lv = ref.quantise(spec, f)
        out[f"quant_{name}_levels"], out[f"quant_{name}_out"] = lv, qf
    out["seed_field_s7"] = ref.seed_random_phase(amp32, 7)  # Rng(7).fork(0) stream
    out["fresnel_q_16x8"] = ref.fresnel_q(16, 8, 532e-9, 0.1, 8e-6, 8e-6)
    np.savez_compressed(os.path.join(HERE, "ref_runs.npz"), **out)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
