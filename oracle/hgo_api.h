/*
 * hgo_api.h — plain-C structs shared by the oracle restatement
 * (hg_oracle.c) and the reference-headers shim (ref_shim.cpp), so one
 * ctypes description in tests/ drives both.  TEST INFRASTRUCTURE ONLY.
 */
#ifndef HGO_API_H
#define HGO_API_H
#include <stdint.h>
#include <stddef.h>

/* Mirrors hologen::SlmSpec (quantise.hpp:20-105). */
typedef struct {
    int mode; /* 0 amplitude, 1 phase (SlmMode, quantise.hpp:14) */
    int levels;
    double min_arg, max_arg;
    int full_circle;
    double min_amp, max_amp;
    const double *illum; /* interleaved complex double, nx*ny, or NULL */
} hgo_slm;


/* Mirrors hologen::IftaConfig (ifta.hpp:29-51) + Freedoms (target.hpp:34-40)
 * + FresnelParams (propagation.hpp:15-32). */
typedef struct {
    int variant;    /* 0 GS, 1 WeightedGS, 2 LiuTaghizadeh (ifta.hpp:18) */
    int iterations;
    uint64_t seed;
    double clamp_lo, clamp_hi, lt_initial_fraction;
    int init_phase; /* 0 Auto, 1 Random, 2 Flat (ifta.hpp:25); 3 = given field */
    int amp_outside_roi, phase_freedom, scale_freedom; /* Freedoms, target.hpp:34-40 */
    int fresnel;
    double wavelength, distance, pitch_x, pitch_y;
    int snapshot_iter; /* >0: copy R (and WGS weights) entering this iteration */
} hgo_ifta_cfg;

#endif
