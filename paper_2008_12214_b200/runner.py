"""Batch executor with device routing: the runner's `batch`
command (src/runner.cpp:365-447) on the GPU through ``hgc_batch_run``.

The reference runs one job per host thread; here jobs that differ only in
seed and target are merged into one batched plan and the groups are spread
over the GPUs (see csrc/batch.cpp).  Each job still reports its own status,
message, final_error and seconds, and ``batch_summary`` renders the same
stdout table and ``batch_summary.csv`` text as cmd_batch (runner.cpp:423-447).
Job discovery from JSON files (the CLI) stays with the reference.
"""
from __future__ import annotations

import ctypes as C
import hashlib
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from ._lib import lib
from .api import _ifta_cfg, _ospr_cfg, _slm
from .types import FresnelParams, IftaConfig, OsprConfig


class HgcBatchJob(C.Structure):
    _fields_ = [("kind", C.c_int), ("ifta", C.c_void_p), ("ospr", C.c_void_p), ("slm", C.c_void_p),
                ("fresnel", C.c_void_p), ("nx", C.c_int), ("ny", C.c_int), ("amplitude", C.c_void_p),
                ("phase", C.c_void_p), ("roi", C.c_void_p), ("levels8", C.c_void_p), ("levels16", C.c_void_p),
                ("trace", C.c_void_p), ("status", C.c_int), ("final_error", C.c_double),
                ("seconds", C.c_double), ("message", C.c_char * 256)]


lib.hgc_batch_run.restype = C.c_int
lib.hgc_batch_run.argtypes = [C.POINTER(HgcBatchJob), C.c_int, C.c_int, C.c_size_t]


@dataclass
class BatchJob:
    """One generate job: an IFTA (optionally Fresnel) or OSPR configuration."""
    name: str
    config: IftaConfig | OsprConfig
    fresnel: FresnelParams | None = None


@dataclass
class BatchRow:
    """runner.cpp BatchRow + the job's results."""
    job: str
    ok: bool = False
    final_error: float = 0.0
    seconds: float = 0.0
    message: str = ""
    levels: np.ndarray | None = None
    trace: np.ndarray | None = field(default=None, repr=False)


def run_batch(jobs: list[BatchJob], max_devices: int = 0, max_group_bytes: int = 0,
              keep_outputs: bool = True) -> list[BatchRow]:
    """Run every job; rows come back in job order (cmd_batch sorts the job
    files first, runner.cpp:377)."""
    rows = [BatchRow(job=j.name) for j in jobs]
    keep: list = []
    roi_pool: dict[bytes, np.ndarray] = {}  # identical ROIs share one buffer so their jobs can batch
    slm_pool: dict[tuple, object] = {}
    arr = (HgcBatchJob * len(jobs))()
    live = []
    for i, (j, row) in enumerate(zip(jobs, rows)):
        cfg = j.config
        try:
            cfg.validate()  # the reference's own validation (ifta.hpp:88, ospr.hpp:70)
        except ValueError as e:
            row.message = str(e)
            continue
        amp = np.ascontiguousarray(cfg.target.amplitude, np.float64)
        ny, nx = amp.shape
        c = arr[i]
        if isinstance(cfg, IftaConfig):
            c.kind = 0
            ic = _ifta_cfg(cfg)
            keep.append(ic)
            c.ifta = C.addressof(ic)
            if j.fresnel is not None:
                fr = _lib.HgcFresnel(j.fresnel.wavelength, j.fresnel.distance, j.fresnel.pixel_pitch_x,
                                     j.fresnel.pixel_pitch_y)
                keep.append(fr)
                c.fresnel = C.addressof(fr)
            if cfg.target.phase is not None:
                ph = np.ascontiguousarray(cfg.target.phase, np.float64)
                keep.append(ph)
                c.phase = ph.ctypes.data
            n_out = nx * ny
            tlen = cfg.iterations
        else:
            c.kind = 1
            oc = _ospr_cfg(cfg)
            keep.append(oc)
            c.ospr = C.addressof(oc)
            n_out = nx * ny * cfg.subframes
            tlen = cfg.subframes
        key = (int(cfg.slm.mode), cfg.slm.levels, cfg.slm.min_arg, cfg.slm.max_arg, bool(cfg.slm.full_circle),
               cfg.slm.min_amp, cfg.slm.max_amp, id(cfg.slm.illumination))
        if key not in slm_pool:
            slm_pool[key] = _slm(cfg.slm, keep)
        c.slm = C.addressof(slm_pool[key])
        c.nx, c.ny = nx, ny
        keep.append(amp)
        c.amplitude = amp.ctypes.data
        if cfg.target.roi is not None:
            r = np.ascontiguousarray(np.asarray(cfg.target.roi) != 0, np.uint8)
            h = hashlib.sha1(r.tobytes()).digest() + bytes(str(r.shape), "ascii")
            c.roi = roi_pool.setdefault(h, r).ctypes.data
        if keep_outputs:
            wide = cfg.slm.levels > 256
            row.levels = np.empty(n_out, np.uint16 if wide else np.uint8)
            row.trace = np.empty(tlen, np.float64)
            if wide:
                c.levels16 = row.levels.ctypes.data
            else:
                c.levels8 = row.levels.ctypes.data
            c.trace = row.trace.ctypes.data
            shape = (cfg.subframes, ny, nx) if c.kind == 1 else (ny, nx)
            row.levels = row.levels.reshape(shape)
        live.append(i)
    keep.append(roi_pool)
    if live:
        sub = (HgcBatchJob * len(live))(*[arr[i] for i in live])
        lib.hgc_batch_run(sub, len(live), max_devices, max_group_bytes)
        for k, i in enumerate(live):
            r, c = rows[i], sub[k]
            r.ok = c.status == _lib.HGC_OK
            r.final_error, r.seconds = c.final_error, c.seconds
            r.message = c.message.decode(errors="replace")
            if not r.ok:
                r.levels = r.trace = None
    return rows


def _fmt9(v: float) -> str:  # runner.cpp:21-25
    return "%#.9g" % v


def batch_summary(rows: list[BatchRow]) -> tuple[str, str]:
    """(stdout table, batch_summary.csv text) as cmd_batch writes them."""
    out = ["%-32s %-8s %16s %10s" % ("job", "status", "final_error", "seconds")]
    csv = "job,status,final_error,seconds,message\n"
    for r in rows:
        if r.ok:
            out.append("%-32s %-8s %16s %10.3f" % (r.job, "ok", _fmt9(r.final_error), r.seconds))
        else:
            out.append("%-32s %-8s %16s %10s" % (r.job, "failed", "-", "-"))
        msg = r.message.replace(",", ";").replace("\n", " ")
        csv += ",".join([r.job, "ok" if r.ok else "failed", _fmt9(r.final_error) if r.ok else "-",
                         _fmt9(r.seconds) if r.ok else "-", msg]) + "\n"
    return "\n".join(out) + "\n", csv
