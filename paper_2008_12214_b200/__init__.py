"""B200-native HoloGen IFTA / OSPR hot path (arXiv 2008.12214).

Gerchberg-Saxton / weighted-GS (Fourier and Fresnel) and One-Step
Phase-Retrieval on hand-written sm_100a kernels behind the C ABI in
include/hologen_b200.h, with the reference's API (proj/include/hologen)
mirrored in Python.  Importing requires the in-tree libhologen_b200.so; there
is no CPU fallback.
"""
from ._lib import HgcError, HgcIOError, HgcUnsupported, exported_symbols
from .api import (IftaPlan, OsprBlockPlan, OsprPlan, Propagator, Quantiser, allowed_states_f32, device_count, fft_forward,
                  fft_inverse, fork_seed, fresnel_forward, fresnel_inverse, make_fresnel_phase, mse, quantise_field,
                  run_adaptive_ospr, run_gs, run_ifta, run_ifta_batch, run_liu_taghizadeh, run_ospr, run_ospr_batch,
                  run_ospr_variant, run_weighted_gs, seed_random_phase, set_device, subframe_mse_statistic,
                  mt_jump_state, run_ifta_f64, run_ospr_f64)
from .types import (PI, TWO_PI, Freedoms, FresnelParams, IftaConfig, IftaVariant, InitPhase, MetricConfig,
                    MetricTrace, Normalization, OsprConfig, OsprRun, OsprVariant, PhaseProfile, RunReport, SlmMode,
                    SlmSpec, SubframeSet, TargetSpec, allowed_states, lt_area_fractions, normalize_image)
from . import io, patterns, runner, shard

__version__ = "0.1.0"
