"""Value types of the reference API (proj/include/hologen/*.hpp), in Python.

Same names, fields, defaults, validation rules and messages as the C++
structs; fields are numpy arrays (row-major ``(ny, nx)``):
complex64 for ``ComplexField<float>``, float64 for ``RealImage``, uint8 for
``RegionMask``.  ``validate()`` raises ``ValueError`` where the reference
throws ``std::invalid_argument``.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

TWO_PI = 6.283185307179586476925286766559
PI = 3.1415926535897932384626433832795


def _require_finite(img, what: str, kind: str = "image") -> None:  # field.hpp:106-115
    if not np.all(np.isfinite(img)):
        raise ValueError(f"{what}: {kind} contains non-finite values")


# ------------------------------------------------------------ quantise.hpp
class SlmMode(IntEnum):  # quantise.hpp:14
    Amplitude = 0
    Phase = 1


@dataclass
class SlmSpec:  # quantise.hpp:20-105
    mode: SlmMode = SlmMode.Phase
    levels: int = 2
    min_arg: float = 0.0
    max_arg: float = 0.0
    full_circle: bool = False
    min_amp: float = 0.0
    max_amp: float = 1.0
    illumination: np.ndarray | None = None  # complex128 (ny, nx)

    @staticmethod
    def phase(levels: int, min_arg: float, max_arg: float) -> "SlmSpec":
        s = SlmSpec(SlmMode.Phase, levels, min_arg, max_arg, False)
        s.validate()
        return s

    @staticmethod
    def full_circle_phase(levels: int, start_arg: float = 0.0) -> "SlmSpec":
        s = SlmSpec(SlmMode.Phase, levels, start_arg, start_arg + TWO_PI, True)
        s.validate()
        return s

    @staticmethod
    def binary_phase() -> "SlmSpec":
        return SlmSpec.phase(2, 0.0, PI)

    @staticmethod
    def amplitude(levels: int, min_amp: float = 0.0, max_amp: float = 1.0) -> "SlmSpec":
        s = SlmSpec(SlmMode.Amplitude, levels, min_amp=min_amp, max_amp=max_amp)
        s.validate()
        return s

    @staticmethod
    def binary_amplitude() -> "SlmSpec":
        return SlmSpec.amplitude(2, 0.0, 1.0)

    def validate(self) -> None:
        if self.levels < 2:
            raise ValueError("SlmSpec: levels must be >= 2")
        if self.mode == SlmMode.Phase:
            if not (math.isfinite(self.min_arg) and math.isfinite(self.max_arg)):
                raise ValueError("SlmSpec: phase range must be finite")
            if not (self.min_arg < self.max_arg) or self.max_arg - self.min_arg > TWO_PI * (1 + 1e-12):
                raise ValueError("SlmSpec: phase range must satisfy min_arg < max_arg <= min_arg + 2*pi")
            if self.full_circle and abs((self.max_arg - self.min_arg) - TWO_PI) > 1e-9:
                raise ValueError("SlmSpec: full_circle requires a 2*pi range")
        else:
            if not (math.isfinite(self.min_amp) and math.isfinite(self.max_amp)):
                raise ValueError("SlmSpec: amplitude range must be finite")
            if not (self.min_amp >= 0) or not (self.min_amp < self.max_amp):
                raise ValueError("SlmSpec: need 0 <= min_amp < max_amp")
        if self.illumination is not None:
            il = np.asarray(self.illumination)
            if not np.all(np.isfinite(il)):
                raise ValueError("SlmSpec: illumination must be finite")
            if np.any(il == 0):
                raise ValueError("SlmSpec: illumination must be nowhere zero")

    def spacing(self) -> float:  # quantise.hpp:99-104
        if self.mode == SlmMode.Phase:
            return TWO_PI / self.levels if self.full_circle else (self.max_arg - self.min_arg) / (self.levels - 1)
        return (self.max_amp - self.min_amp) / (self.levels - 1)


def allowed_states(spec: SlmSpec) -> np.ndarray:  # quantise.hpp:111-124
    spec.validate()
    spac = spec.spacing()
    k = np.arange(spec.levels, dtype=np.float64)
    if spec.mode == SlmMode.Phase:
        a = spec.min_arg + k * spac
        return np.cos(a) + 1j * np.sin(a)
    return (spec.min_amp + k * spac).astype(np.complex128)


# ---------------------------------------------------------- propagation.hpp
@dataclass
class FresnelParams:  # propagation.hpp:15-32
    wavelength: float = 0.0
    distance: float = 0.0
    pixel_pitch_x: float = 0.0
    pixel_pitch_y: float = 0.0

    def validate(self) -> None:
        if not (self.wavelength > 0) or not math.isfinite(self.wavelength):
            raise ValueError("FresnelParams: wavelength must be positive")
        if self.distance == 0 or not math.isfinite(self.distance):
            raise ValueError("FresnelParams: distance must be non-zero")
        if (not (self.pixel_pitch_x > 0) or not (self.pixel_pitch_y > 0) or not math.isfinite(self.pixel_pitch_x)
                or not math.isfinite(self.pixel_pitch_y)):
            raise ValueError("FresnelParams: pixel pitches must be positive")


# --------------------------------------------------------------- target.hpp
class Normalization(IntEnum):  # target.hpp:13
    MaxToOne = 0
    UnitEnergy = 1


def normalize_image(img: np.ndarray, norm: Normalization) -> np.ndarray:  # target.hpp:15-30
    """In place (like the reference) and returned for convenience."""
    if norm == Normalization.MaxToOne:
        acc = float(np.max(img)) if img.size else 0.0
        acc = max(acc, 0.0)
        if acc == 0.0:
            return img
        img *= 1.0 / acc
        return img
    flat = img.ravel()
    sq = flat * flat
    acc = float(np.add.accumulate(sq)[-1]) if sq.size else 0.0  # the reference's sequential sum, bit for bit
    if acc <= 0.0:
        raise ValueError("normalize_image: zero-energy image cannot be energy-normalized")
    img *= math.sqrt(img.size / acc)
    return img


@dataclass
class Freedoms:  # target.hpp:34-40
    amplitude_outside_roi: bool = False
    phase: bool = True
    scale: bool = False


@dataclass
class TargetSpec:  # target.hpp:45-73
    amplitude: np.ndarray = field(default_factory=lambda: np.zeros((0, 0)))
    phase: np.ndarray | None = None  # turns in [0, 1)
    roi: np.ndarray | None = None  # uint8 mask
    freedoms: Freedoms = field(default_factory=Freedoms)

    def width(self) -> int:
        return int(self.amplitude.shape[1])

    def height(self) -> int:
        return int(self.amplitude.shape[0])

    def validate(self) -> None:
        a = np.asarray(self.amplitude)
        if a.ndim != 2 or a.shape[0] <= 0 or a.shape[1] <= 0:
            raise ValueError("TargetSpec: amplitude image is empty")
        _require_finite(a, "TargetSpec.amplitude")
        if np.any(a < 0):
            raise ValueError("TargetSpec: amplitude must be non-negative")
        if self.phase is not None:
            if np.asarray(self.phase).shape != a.shape:
                raise ValueError("TargetSpec: phase dimensions mismatch")
            _require_finite(self.phase, "TargetSpec.phase")
        if self.roi is not None:
            if np.asarray(self.roi).shape != a.shape:
                raise ValueError("TargetSpec: roi dimensions mismatch")
            if not np.any(np.asarray(self.roi) != 0):
                raise ValueError("TargetSpec: roi covers no pixels")


# ----------------------------------------------------------------- ifta.hpp
class IftaVariant(IntEnum):  # ifta.hpp:18
    GS = 0
    WeightedGS = 1
    LiuTaghizadeh = 2


class InitPhase(IntEnum):  # ifta.hpp:25 (+ Given: start from a supplied replay field)
    Auto = 0
    Random = 1
    Flat = 2
    Given = 3


class LtGrowth(IntEnum):  # ifta.hpp:27
    Linear = 0


@dataclass
class IftaConfig:  # ifta.hpp:29-51
    variant: IftaVariant = IftaVariant.GS
    iterations: int = 1
    slm: SlmSpec = field(default_factory=SlmSpec)
    target: TargetSpec = field(default_factory=TargetSpec)
    seed: int = 0
    weight_clamp_lo: float = 0.1
    weight_clamp_hi: float = 10.0
    lt_initial_fraction: float = 0.1
    lt_growth: LtGrowth = LtGrowth.Linear
    init_phase: InitPhase = InitPhase.Auto

    def validate(self) -> None:
        if self.iterations < 1:
            raise ValueError("IftaConfig: iterations must be >= 1")
        if not (self.weight_clamp_lo > 0) or not (self.weight_clamp_hi >= self.weight_clamp_lo):
            raise ValueError("IftaConfig: weight clamp bounds invalid")
        if not (self.lt_initial_fraction > 0) or not (self.lt_initial_fraction <= 1):
            raise ValueError("IftaConfig: lt_initial_fraction must be in (0,1]")
        self.slm.validate()
        self.target.validate()


def lt_area_fractions(iterations: int, initial_fraction: float) -> list[float]:  # ifta.hpp:55-63
    if iterations < 1:
        raise ValueError("lt_area_fractions: iterations must be >= 1")
    a = [0.0] * iterations
    for k in range(1, iterations):
        a[k - 1] = initial_fraction + (1.0 - initial_fraction) * (k - 1) / (iterations - 1)
    a[iterations - 1] = 1.0
    return a


# ----------------------------------------------------------------- ospr.hpp
class OsprVariant(IntEnum):  # ospr.hpp:18
    Ospr = 0
    AdaptiveOspr = 1


@dataclass
class OsprConfig:  # ospr.hpp:20-38
    variant: OsprVariant = OsprVariant.Ospr
    subframes: int = 1
    slm: SlmSpec = field(default_factory=SlmSpec)
    target: TargetSpec = field(default_factory=TargetSpec)
    seed: int = 0
    feedback_gain: float = 1.0

    def validate(self) -> None:
        if self.subframes < 1:
            raise ValueError("OsprConfig: subframes must be >= 1")
        if not (0.0 <= self.feedback_gain <= 1.0):
            raise ValueError("OsprConfig: feedback_gain must be in [0,1]")
        self.slm.validate()
        self.target.validate()


# --------------------------------------------------------------- report.hpp
@dataclass
class MetricTrace:  # report.hpp:24-35
    name: str = "metric"
    points: list = field(default_factory=list)

    def append(self, iteration: int, value: float) -> None:
        if self.points and iteration <= self.points[-1][0]:
            raise ValueError("MetricTrace: iterations must be strictly increasing")
        self.points.append((int(iteration), float(value)))

    def size(self) -> int:
        return len(self.points)

    def values(self) -> np.ndarray:
        return np.array([v for _, v in self.points], dtype=np.float64)


@dataclass
class PhaseProfile:  # report.hpp:38-45
    transform: float = 0.0
    constraint: float = 0.0
    metric: float = 0.0
    other: float = 0.0

    def total(self) -> float:
        return self.transform + self.constraint + self.metric + self.other


@dataclass
class RunReport:  # report.hpp:48-65 (+ levels: the hologram's level indices)
    algorithm: str = ""
    seed: int = 0
    hologram: np.ndarray | None = None
    replay: np.ndarray | None = None
    trace: MetricTrace = field(default_factory=MetricTrace)
    extra_traces: list = field(default_factory=list)
    final_error: float = 0.0
    seconds: float = 0.0
    profile: PhaseProfile = field(default_factory=PhaseProfile)
    evaluations: int = 0
    accepted: int = 0
    decisions: list = field(default_factory=list)
    levels: np.ndarray | None = None
    weights: np.ndarray | None = None  # WGS weights of a checkpointed run (run_ifta(..., checkpoint=True))
    efficiency: float | None = None  # extension: diffraction efficiency of the final replay (hgc_ifta_io::efficiency)


@dataclass
class SubframeSet:  # ospr.hpp:42-47 (frames: (N, ny, nx) complex64)
    frames: np.ndarray | None = None
    mean_intensity: np.ndarray | None = None
    per_frame_mse: list = field(default_factory=list)
    levels: np.ndarray | None = None


@dataclass
class OsprRun:  # ospr.hpp:49-53
    set: SubframeSet = field(default_factory=SubframeSet)
    report: RunReport = field(default_factory=RunReport)


@dataclass
class MetricConfig:  # metrics.hpp:19-38 (MSE, phase-insensitive on the GPU path)
    kind: str = "mse"
    phase_sensitive: bool = False
    mask: np.ndarray | None = None
    scale_free: bool = False
