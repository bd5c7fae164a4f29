/*
 * hologen_b200.h — C ABI of the B200-native HoloGen IFTA / OSPR hot path.
 *
 * This is the drop-in boundary.  Each entry point replaces one reference
 * interface (paths relative to /root/reference/proj/include/hologen/):
 *
 *   hgc_ifta_run           run_gs / run_weighted_gs / run_liu_taghizadeh /
 *                          run_ifta<float>            ifta.hpp:239-263
 *                          (detail::run_ifta           ifta.hpp:86-235),
 *                          batched over targets like cmd_batch
 *                          (src/runner.cpp:365-421)
 *   hgc_ospr_run           run_ospr / run_adaptive_ospr /
 *                          run_ospr_variant<float>     ospr.hpp:168-185
 *                          (detail::run_ospr_impl      ospr.hpp:68-164),
 *                          batched over independent jobs
 *   hgc_fft2d              FftBackend<float>::forward / inverse
 *                          fft.hpp:17-27 (FftwBackend::run,
 *                          src/fftw_backend.cpp:113-124)
 *   hgc_propagate          Propagator<float>::forward / inverse
 *                          propagation.hpp:60-116
 *   hgc_quantise           Quantiser<float>::apply      quantise.hpp:208-216
 *                          (quantise_field              quantise.hpp:234-243)
 *   hgc_seed_random_phase  seed_random_phase<float>     rng.hpp:54-67
 *   hgc_mse                mse (phase-insensitive)      metrics.hpp:70-124
 *   hgc_fresnel_phase      make_fresnel_phase<float>    propagation.hpp:36-54
 *   hgc_subframe_mse_statistic  subframe_mse_statistic  ospr.hpp:58-64
 *
 * Conventions (field.hpp:27-66): fields are row-major data[y*nx + x];
 * complex values are interleaved float pairs (layout-compatible with
 * std::complex<float>); target images are double; masks are uint8.  All
 * pointers passed to hgc_*_run / primitives are HOST pointers owned by the
 * caller; the library owns device memory.  The plan API (hgc_*_plan_*) keeps
 * inputs and outputs resident in HBM for repeated execution.
 *
 * Errors: every function returns HGC_OK (0) or an hgc_status; the message is
 * in hgc_last_error() (thread-local).  HGC_EINVAL corresponds to the
 * reference's std::invalid_argument (same messages), HGC_ECUDA / HGC_EUNSUPPORTED
 * to std::runtime_error.  There is no CPU fallback: sizes the GPU path does
 * not support (non powers of two, > 4096 per side) fail with HGC_EUNSUPPORTED.
 *
 * Threading (fft.hpp:79-83, runner.cpp:387-421): every call is re-entrant;
 * each call / plan uses its own CUDA stream on the calling thread's current
 * device (hgc_set_device).
 */
#ifndef HOLOGEN_B200_H
#define HOLOGEN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HGC_ABI_VERSION 5

typedef enum {
    HGC_OK = 0,
    HGC_EINVAL = 1,       /* std::invalid_argument in the reference */
    HGC_ECUDA = 2,        /* device / runtime failure */
    HGC_EUNSUPPORTED = 3, /* valid for the reference, outside the GPU path's scope */
    HGC_EIO = 4           /* file / format error: std::runtime_error in the reference (io.cpp:16) */
} hgc_status;

/* hologen::SlmSpec (quantise.hpp:20-105).  mode: 0 Amplitude, 1 Phase.
 * illumination: NULL or interleaved complex<double> [ny][nx]. */
typedef struct hgc_slm {
    int mode;
    int levels;
    double min_arg;
    double max_arg;
    int full_circle;
    double min_amp;
    double max_amp;
    const double* illumination;
} hgc_slm;

/* hologen::FresnelParams (propagation.hpp:15-32). */
typedef struct hgc_fresnel {
    double wavelength;
    double distance;
    double pixel_pitch_x;
    double pixel_pitch_y;
} hgc_fresnel;

/* hologen::IftaConfig (ifta.hpp:29-51) + TargetSpec::freedoms (target.hpp:34-40).
 * variant: 0 GS, 1 WeightedGS, 2 LiuTaghizadeh.
 * init_phase: 0 Auto, 1 Random, 2 Flat, 3 Given (extension: start from
 * hgc_ifta_io.init_field, e.g. to resume from a checkpointed replay field). */
typedef struct hgc_ifta_cfg {
    int variant;
    int iterations;
    uint64_t seed;
    double weight_clamp_lo;
    double weight_clamp_hi;
    double lt_initial_fraction;
    int init_phase;
    int freedom_amplitude_outside_roi;
    int freedom_phase;
    int freedom_scale;
} hgc_ifta_cfg;

/* Inputs and outputs of one batched IFTA call.  batch targets share size,
 * SLM, propagation and ROI.  Any output pointer may be NULL. */
typedef struct hgc_ifta_io {
    const double* amplitude;    /* TargetSpec::amplitude  [batch][ny][nx] */
    const double* phase;        /* TargetSpec::phase (turns) [batch][ny][nx] or NULL */
    const uint8_t* roi;         /* TargetSpec::roi [ny][nx] or NULL */
    const uint64_t* seeds;      /* [batch] IftaConfig::seed per target, or NULL = cfg->seed */
    const float* init_field;    /* init_phase == 3: complex [batch][ny][nx] */
    const float* init_weights;  /* init_phase == 3, WGS: [batch][ny][nx] or NULL (= 1) */
    float* hologram;            /* RunReport::hologram  complex [batch][ny][nx] */
    uint8_t* levels8;           /* level indices of the hologram (levels <= 256) */
    uint16_t* levels16;         /* level indices (any level count <= 65536) */
    float* replay;              /* RunReport::replay    complex [batch][ny][nx] */
    double* trace;              /* RunReport::trace     [batch][iterations] */
    double* final_error;        /* RunReport::final_error [batch] */
    double* seconds;            /* RunReport::seconds (whole call) */
    const float* fresnel_q;     /* optional complex [ny][nx] quadratic phase Q to use instead of
                                   computing it from hgc_fresnel (e.g. taken from an existing
                                   Propagator<float>, propagation.hpp:97-103) */
    /* Output encodings computed on the device from the resident results
     * (the runner's hologram.png / replay.png, runner.cpp:251-266): */
    uint8_t* hologram_gray8;    /* write_hologram_png pixels lround(255 k / (L-1)) [batch][ny][nx],
                                   L <= 256 (io.cpp:272-287) */
    uint8_t* replay_gray8;      /* write_replay_png pixels [batch][ny][nx] (io.cpp:189-205) */
    double* replay_peak;        /* its amplitude_at_255 [batch] (io.cpp:206-207) */
    uint8_t* levels1;           /* 2-level SLMs: the levels as bit-planes, bit (i & 7) of byte i >> 3 of
                                   each target's row-major plane [batch][ny*nx/8] (binary SLM frames) */
    /* Checkpoint (extension; the state a resumed run starts from): nonzero =
     * the last iteration also applies the replay-plane constraint (ifta.hpp:185-224,
     * incl. the WGS weight update and the LT rectangle of iteration K), so
     * `replay` receives the constrained field R_K instead of the unconstrained
     * one and `weights` the WGS weights W_K.  For GS and WGS, running K1
     * iterations with checkpoint and then K2 with init_phase Given from
     * (replay, weights) reproduces a K1 + K2 run bit for bit (LT's schedule
     * depends on K).  trace / levels / hologram are unchanged. */
    int checkpoint;
    float* weights;             /* WGS weights after the run [batch][ny][nx] (1 for other variants) */
    /* RunReport::profile (report.hpp:38-45): {transform, constraint, metric,
     * other} seconds of hgc_ifta_run, attributed from per-pass device times
     * (DESIGN.md §5); their sum equals *seconds.  Only hgc_ifta_run fills it. */
    double* profile;
    /* Diffraction efficiency of the final replay (extension; the reference has
     * no efficiency metric): the replay power on the target's support (T > 0,
     * inside the ROI when one is given) over the total replay power,
     * sum_{T>0, roi} |R|^2 / sum |R|^2, reduced in the last iteration's fused
     * column pass.  [batch] */
    double* efficiency;
} hgc_ifta_io;

/* hologen::OsprConfig (ospr.hpp:20-38).  variant: 0 Ospr, 1 AdaptiveOspr.
 * freedom_scale: TargetSpec::freedoms.scale (scale-free MSE). */
typedef struct hgc_ospr_cfg {
    int variant;
    int subframes;
    uint64_t seed;
    double feedback_gain;
    int freedom_scale;
} hgc_ospr_cfg;

/* One batched OSPR call over `jobs` independent runs (one seed each). */
typedef struct hgc_ospr_io {
    const double* amplitude;    /* [ny][nx] shared by all jobs, or [jobs][ny][nx] */
    int per_job_target;         /* 0: amplitude shared, 1: one target per job */
    const uint8_t* roi;         /* [ny][nx] or NULL */
    const uint64_t* seeds;      /* [jobs] or NULL = cfg->seed */
    uint8_t* levels8;           /* SubframeSet::frames as levels [jobs][subframes][ny][nx] */
    uint16_t* levels16;
    float* frames;              /* SubframeSet::frames complex [jobs][subframes][ny][nx] */
    double* frame_mse;          /* SubframeSet::per_frame_mse [jobs][subframes] */
    double* cumulative_mse;     /* RunReport::trace "cumulative_mse" [jobs][subframes] */
    double* mean_intensity;     /* SubframeSet::mean_intensity [jobs][ny][nx] */
    float* replay;              /* RunReport::replay complex [jobs][ny][nx] */
    double* final_error;        /* [jobs] */
    double* seconds;
    /* device-side output encodings, as hgc_ifta_io: */
    uint8_t* frames_gray8;      /* frame levels as write_hologram_png pixels [jobs][subframes][ny][nx] */
    uint8_t* replay_gray8;      /* write_replay_png pixels of the replay [jobs][ny][nx] */
    double* replay_peak;        /* [jobs] */
    uint8_t* levels1;           /* 2-level SLMs: frame levels as bit-planes [jobs][subframes][ny*nx/8],
                                   bit (i & 7) of byte i >> 3 (what a binary FLC SLM is fed) */
    double* profile;            /* RunReport::profile {transform, constraint, metric, other} of
                                   hgc_ospr_run (as hgc_ifta_io::profile) or NULL */
} hgc_ospr_io;

/* ------------------------------------------------------------ library */
int hgc_abi_version(void);
const char* hgc_last_error(void);
int hgc_device_count(int* count);
int hgc_set_device(int device);
/* Device routing for callers that run jobs on their own host threads (the
 * runner's batch pool, runner.cpp:387-421, via the C++ drop-in; SURVEY §8
 * b5/f2): policy 1 binds each host thread, at its first hgc_ifta_run /
 * hgc_ospr_run, to the next device round-robin (job thread i -> GPU i mod G);
 * policy 0 (default) uses the thread's current device. */
int hgc_set_device_policy(int policy);
/* Largest supported power-of-two side length (4096). */
int hgc_max_side(void);

/* ------------------------------------------------- algorithm entry points */
int hgc_ifta_run(const hgc_ifta_cfg* cfg, const hgc_slm* slm, const hgc_fresnel* fresnel,
                 int nx, int ny, int batch, hgc_ifta_io* io);
int hgc_ospr_run(const hgc_ospr_cfg* cfg, const hgc_slm* slm, int nx, int ny, int jobs,
                 hgc_ospr_io* io);
/* Fresnel OSPR (extension; the reference rejects OSPR + Fresnel,
 * src/config.cpp:443-445): the subframe loop of run_ospr_impl with the
 * Propagator<float> inverse / forward (propagation.hpp:81-95) in place of the
 * bare FFTs: f = IFFT(seed) conj(Q), quantise, R = FFT(f Q).  fresnel == NULL
 * is hgc_ospr_run.  Parity is pinned only against a composed oracle. */
int hgc_ospr_run_fresnel(const hgc_ospr_cfg* cfg, const hgc_slm* slm, const hgc_fresnel* fresnel, int nx, int ny,
                         int jobs, hgc_ospr_io* io);

/* ------------------------------------------ device-resident plan API */
typedef struct hgc_ifta_plan hgc_ifta_plan;
typedef struct hgc_ospr_plan hgc_ospr_plan;

int hgc_ifta_plan_create(hgc_ifta_plan** plan, const hgc_ifta_cfg* cfg, const hgc_slm* slm,
                         const hgc_fresnel* fresnel, int nx, int ny, int batch);
/* Host->device copy of io's inputs (amplitude, phase, roi, seeds, init_*),
 * asynchronous on the plan's stream: with pinned host buffers it returns once
 * the copies are enqueued, so the caller must keep them unchanged until the
 * next execute has completed (download returned).  TargetSpec validation
 * (target.hpp:52-73) runs on the device; its error (HGC_EINVAL, same message)
 * is returned by the next download.  hgc_ifta_run validates eagerly. */
int hgc_ifta_plan_upload(hgc_ifta_plan* plan, const hgc_ifta_io* io);
/* Enqueue one full run (init + iterations + trace reduction) on `stream`
 * (a cudaStream_t, or NULL for the plan's own stream).  Asynchronous. */
int hgc_ifta_plan_execute(hgc_ifta_plan* plan, void* stream);
/* Wait for this plan's last execute and copy io's requested outputs to the
 * host (HGC_EINVAL if the uploaded target failed validation). */
int hgc_ifta_plan_download(hgc_ifta_plan* plan, hgc_ifta_io* io);
/* Device pointers of the resident buffers (any may be NULL on input):
 * field = replay after execute (complex float [batch][ny][nx]),
 * levels = uint8 or uint16 [batch][ny][nx], trace = double [batch][iterations]. */
int hgc_ifta_plan_device_ptrs(hgc_ifta_plan* plan, void** field, void** levels, void** trace);
/* Kernel launches one execute enqueues. */
int hgc_ifta_plan_launches(hgc_ifta_plan* plan);
/* Average device time (ms) of the seed kernel, the fused row pass and the
 * fused column pass, each launched `reps` times on the plan's stream (CUDA
 * events).  Advances the resident state: call after the timed work. */
int hgc_ifta_plan_profile(hgc_ifta_plan* plan, int reps, double* ms_seed, double* ms_row, double* ms_col);
/* Per-pass device time inside the plan's own graph: with timing on (set
 * before the first execute), CUDA events are recorded around the first target
 * group's row and column passes of every iteration; kernel_times returns
 * their average over iterations 1..K-1 of the last execute (ms) and that
 * count.  Measurement support, not part of the reference interface. */
int hgc_ifta_plan_set_kernel_timing(hgc_ifta_plan* plan, int on);
int hgc_ifta_plan_kernel_times(hgc_ifta_plan* plan, double* ms_row, double* ms_col, int* iterations);
int hgc_ifta_plan_destroy(hgc_ifta_plan* plan);

int hgc_ospr_plan_create(hgc_ospr_plan** plan, const hgc_ospr_cfg* cfg, const hgc_slm* slm, int nx,
                         int ny, int jobs, int per_job_target);
/* Asynchronous as hgc_ifta_plan_upload (validation errors on download). */
int hgc_ospr_plan_upload(hgc_ospr_plan* plan, const hgc_ospr_io* io);
int hgc_ospr_plan_execute(hgc_ospr_plan* plan, void* stream);
int hgc_ospr_plan_download(hgc_ospr_plan* plan, hgc_ospr_io* io);
/* levels = uint8/uint16 [jobs][subframes][ny][nx]; traces = double
 * [jobs][subframes][2] (frame mse, cumulative mse); intensity = float [jobs][ny][nx]. */
int hgc_ospr_plan_device_ptrs(hgc_ospr_plan* plan, void** levels, void** traces, void** intensity);
int hgc_ospr_plan_launches(hgc_ospr_plan* plan);
/* Average device time (ms) of one subframe's seed / inverse-column / fused
 * row / accumulating-column passes (CUDA events, `reps` launches each). */
int hgc_ospr_plan_profile(hgc_ospr_plan* plan, int reps, double* ms_seed, double* ms_col_inv, double* ms_row,
                          double* ms_col_acc);
int hgc_ospr_plan_destroy(hgc_ospr_plan* plan);
/* The plan's propagation: Fresnel (hgc_ospr_run_fresnel) or NULL = Fourier.
 * Before the first execute. */
int hgc_ospr_plan_set_fresnel(hgc_ospr_plan* plan, const hgc_fresnel* fresnel);

/* Subframe-block sharding of ONE plain OSPR job across ranks (
 * the loop of run_ospr_impl, ospr.hpp:105-147, split at subframe
 * boundaries).  The plan computes global subframes [first, first + count) of
 * the cfg->subframes-frame job: its random-phase stream starts first*npix
 * draws into Rng(seed).fork(0) (ospr.hpp:89, :118) by jump-ahead, so frames,
 * levels and frame MSEs are those of the unsharded run.  Upload / execute /
 * download as for hgc_ospr_plan_* with jobs = 1; traces/levels hold the
 * block's `count` frames.  Adaptive OSPR is sequential: HGC_EUNSUPPORTED.
 *
 * Exchange: hgc_ospr_block_sum gives this block's intensity sum B (float
 * device buffer, `count` elements, plan layout) after execute; all-gather the
 * B of every block in block order into one device buffer [nblocks][count]
 * (e.g. ncclAllGather), then hgc_ospr_block_finish computes the block's
 * cumulative MSEs (ospr.hpp:142-145) from the prefix of the earlier blocks
 * and sets the intensity to the job total (mean_intensity / replay of the
 * whole job on download). */
int hgc_ospr_block_plan_create(hgc_ospr_plan** plan, const hgc_ospr_cfg* cfg, const hgc_slm* slm, int nx, int ny,
                               int first, int count);
int hgc_ospr_block_sum(hgc_ospr_plan* plan, void** dev_ptr, size_t* count);
int hgc_ospr_block_finish(hgc_ospr_plan* plan, const void* gathered, int nblocks, int index, void* stream);

/* --------------------------------------- f64 loops */
/* run_ifta<double> / run_ospr_variant<double> (ifta.hpp:86-235,
 * ospr.hpp:68-185) on the device, one target per call: the reference's
 * double arithmetic per pixel (quantiser decisions, constraint, MSE, OSPR
 * accumulation; no FMA contraction), double transforms of any size (as
 * hgc_fft2d_f64), seeds from the same Rng(seed).fork(0) stream.  Complex
 * buffers are interleaved double [ny][nx] (std::complex<double>). */
typedef struct hgc_ifta_io64 {
    const double* amplitude;    /* TargetSpec::amplitude [ny][nx] */
    const double* phase;        /* TargetSpec::phase (turns) or NULL */
    const uint8_t* roi;         /* or NULL */
    const double* init_field;   /* init_phase == 3: complex [ny][nx] */
    const double* init_weights; /* init_phase == 3, WGS, or NULL */
    double* hologram;           /* RunReport::hologram complex [ny][nx] */
    double* replay;             /* RunReport::replay complex [ny][nx] */
    int32_t* levels;            /* level indices [ny][nx] */
    double* trace;              /* [iterations] */
    double* final_error;
    const double* fresnel_q;    /* optional complex [ny][nx] Q to use instead of computing it from
                                   hgc_fresnel (e.g. from a Propagator<double>, propagation.hpp:97-103) */
    double* profile;            /* RunReport::profile {transform, constraint, metric, other} seconds:
                                   device time of each reference phase (ifta.hpp:166-226), other =
                                   the rest of the call, or NULL */
} hgc_ifta_io64;
int hgc_ifta_run_f64(const hgc_ifta_cfg* cfg, const hgc_slm* slm, const hgc_fresnel* fresnel, int nx, int ny,
                     hgc_ifta_io64* io);
typedef struct hgc_ospr_io64 {
    const double* amplitude;    /* [ny][nx] */
    const uint8_t* roi;
    double* frames;             /* complex [subframes][ny][nx] */
    int32_t* levels;            /* [subframes][ny][nx] */
    double* frame_mse;          /* [subframes] */
    double* cumulative_mse;     /* [subframes] */
    double* mean_intensity;     /* [ny][nx] */
    double* replay;             /* complex [ny][nx] */
    double* final_error;
    double* profile;            /* RunReport::profile as hgc_ifta_io64 (ospr.hpp:105-147 phases), or NULL */
} hgc_ospr_io64;
int hgc_ospr_run_f64(const hgc_ospr_cfg* cfg, const hgc_slm* slm, int nx, int ny, hgc_ospr_io64* io);

/* ------------------------------ batch executor */
/* One job of the runner's `batch` command (runner.cpp:365-421): a generate
 * run of one target.  Inputs are caller-owned host buffers; the outputs
 * (levels, trace) are optional.  status / message / final_error / seconds
 * are filled per job like cmd_batch's BatchRow. */
typedef struct hgc_batch_job {
    int kind;                    /* 0 IFTA (ifta), 1 OSPR (ospr) */
    const hgc_ifta_cfg* ifta;
    const hgc_ospr_cfg* ospr;
    const hgc_slm* slm;
    const hgc_fresnel* fresnel;  /* IFTA Fresnel propagation, or NULL */
    int nx, ny;
    const double* amplitude;     /* [ny][nx] */
    const double* phase;         /* IFTA target phase or NULL */
    const uint8_t* roi;          /* [ny][nx] or NULL */
    uint8_t* levels8;            /* IFTA [ny][nx]; OSPR [subframes][ny][nx] (levels <= 256) */
    uint16_t* levels16;
    double* trace;               /* IFTA mse [iterations]; OSPR cumulative mse [subframes] */
    int status;                  /* hgc_status of this job */
    double final_error;
    double seconds;              /* wall time of the batched group that ran this job */
    char message[256];           /* error message when status != HGC_OK */
} hgc_batch_job;
/* Runs every job.  Jobs whose configurations differ only in seed and target
 * share one batched plan (one CUDA graph for the group); groups are spread
 * over min(max_devices, device count) GPUs (max_devices <= 0: all), one host
 * thread per device, largest groups first onto the least-loaded device.
 * max_group_bytes caps a group's resident footprint (0: 16 GiB).  A failing
 * group is re-run job by job so each failure stays with its own job.
 * Returns HGC_OK if every job succeeded, else the first failing job's status. */
int hgc_batch_run(hgc_batch_job* jobs, int njobs, int max_devices, size_t max_group_bytes);

/* --------------------------------- output formats */
/* write_field_dump (io.cpp:168-186): HGF1 = "HGF1", u32 nx, u32 ny, u8
 * precision (4 float / 8 double), then interleaved little-endian (re, im).
 * Non-finite values: HGC_EINVAL "field dump: field contains non-finite values". */
int hgc_write_field_dump(const char* path, int nx, int ny, int precision, const void* data);
/* read_field_dump (io.cpp:316-345), same checks and messages (HGC_EIO).
 * data == NULL: validate the file and return nx, ny, precision only. */
int hgc_read_field_dump(const char* path, int* nx, int* ny, int* precision, void* data);
/* write_hologram_png's pixel encoding lround(255 k / (L-1)) (io.cpp:272-287) and
 * read_hologram_png's inverse (io.cpp:289-298), with their validation. */
int hgc_levels_to_gray8(const int32_t* levels, int width, int height, int level_count, uint8_t* out);
int hgc_gray8_to_levels(const uint8_t* px, size_t n, int level_count, int32_t* out);
/* write_replay_png's pixels on the device (io.cpp:189-205): amp = |z| in
 * double, peak = max amp, px = clamp(lround(amp * 255 / peak)), 0 if peak == 0. */
int hgc_replay_to_gray8(const float* replay, int nx, int ny, int batch, uint8_t* out, double* peak);
/* The "<png_path>.scale.txt" companion: "amplitude_at_255=<shortest double>\n". */
int hgc_write_replay_scale(const char* png_path, double peak);
/* write_png_gray (io.cpp:221-237): an 8-bit greyscale PNG (zlib deflate; the
 * reference uses libpng's simplified API).  HGC_EINVAL "write_png_gray: pixel
 * buffer does not match dimensions", HGC_EIO on file errors. */
int hgc_write_png_gray(const char* path, const uint8_t* pixels, int width, int height);
/* read_png_gray8 (io.cpp:239-258) for 8-bit greyscale PNGs: pixels == NULL
 * returns the size only.  HGC_EIO "not a PNG file: <path>" / "png decode failed (...)". */
int hgc_read_png_gray8(const char* path, int* width, int* height, uint8_t* pixels);

/* ------------------------------------------------------- primitives */
/* Unitary 2-D DFT of `batch` fields, sign -1 forward / +1 inverse; in == out
 * allowed.  Any nx, ny >= 1 like FftBackend (fft.hpp:17-27): powers of two
 * up to 4096 on the fused float kernels, other lengths up to 2048 by
 * Bluestein's algorithm in double (rounded back to float). */
int hgc_fft2d(int nx, int ny, int sign, int batch, const float* in, float* out);
/* The same for complex128 (FftBackend<double>, fft.hpp:17-27):
 * double-precision butterflies and twiddles, scale 1/sqrt(nx*ny) in double. */
int hgc_fft2d_f64(int nx, int ny, int sign, int batch, const double* in, double* out);
/* Propagator<float>::forward (sign -1: FFT(f*Q)) / inverse (sign +1:
 * IFFT(F)*conj(Q)), propagation.hpp:81-95; fresnel == NULL is the Fourier
 * propagator (= hgc_fft2d). */
int hgc_propagate(int nx, int ny, int sign, const hgc_fresnel* fresnel, int batch, const float* in, float* out);
/* Snap every pixel of `batch` fields in place; levels (int32, may be NULL). */
int hgc_quantise(const hgc_slm* slm, int nx, int ny, int batch, float* field, int32_t* levels);
/* seed_random_phase<float>(amp, Rng) with the engine seeded by
 * `engine_seed` (Rng(seed).fork(0) uses hgc_fork_seed(seed, 0)) after
 * discarding `skip` draws (std::mt19937_64::discard, by jump-ahead: O(1) in
 * skip).  The draws are split across CTAs by jump-ahead; the result is the
 * single sequential stream of rng.hpp:54-67. */
/* Host utility: the std::mt19937_64 (rng.hpp:23-34) state after `draws`
 * draws from seed `engine_seed`, as the 312 raw words x_draws .. x_draws+311
 * whose twist yields the next output (libstdc++ _M_x with _M_p == 312).
 * Computed by jump-ahead (x^(draws-1) mod the engine's characteristic
 * polynomial); no device needed. */
int hgc_mt_jump_state(uint64_t engine_seed, uint64_t draws, uint64_t* window);
int hgc_seed_random_phase(const double* amplitude, int nx, int ny, uint64_t engine_seed,
                          uint64_t skip, float* out);
uint64_t hgc_fork_seed(uint64_t seed, uint64_t stream);
/* Synthetic targets (host, no device): patterns::smooth_blobs (patterns.hpp:55-80,
 * peak-normalised) and normalize_image (target.hpp:15-30; unit_energy 0 =
 * MaxToOne, 1 = UnitEnergy; HGC_EINVAL for a zero-energy image), bit-identical
 * to the reference's (same operation order, the C library's exp). */
int hgc_smooth_blobs(int width, int height, double* out);
int hgc_normalize_image(double* img, size_t n, int unit_energy);
/* mse(target, replay, {mask, scale_free}) phase-insensitive. */
int hgc_mse(const double* target, const float* replay, const uint8_t* mask, int nx, int ny,
            int scale_free, double* out);
int hgc_fresnel_phase(int nx, int ny, const hgc_fresnel* params, float* q);
double hgc_subframe_mse_statistic(const double* per_frame_mse, int n);

#ifdef __cplusplus
}
#endif
#endif /* HOLOGEN_B200_H */
