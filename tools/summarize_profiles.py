"""Turn gpurun_out/ ncu artefacts into committed summaries under profiles/.
  python tools/summarize_profiles.py <round tag>"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G = os.path.join(ROOT, "gpurun_out")
P = os.path.join(ROOT, "profiles")
tag = sys.argv[1] if len(sys.argv) > 1 else "r01"

# 1. launch list (per-launch device time, serialized/cold under ncu)
rows = list(csv.reader(open(os.path.join(G, "launches.csv"))))
hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value")
per = collections.defaultdict(list)
for r in rows[hdr_i + 1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        name = r[ki].split("(")[0].replace("void ", "")
        per[name].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in per.values())
lines = [f"# ncu launch list of `python bench.py --steps 2 --warmup 1 --no-cpu --no-e2e` (first 400 launches)",
         "# --metrics gpu__time_duration.sum --clock-control none; cold-cache & serialised: compare shares",
         f"{'kernel':60s} {'launches':>8s} {'mean_us':>10s} {'share':>7s}"]
for name, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
    lines.append(f"{name[:60]:60s} {len(v):8d} {sum(v) / len(v) / 1e3:10.1f} {sum(v) / tot:7.3f}")
open(os.path.join(P, f"{tag}_launches.txt"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))

# 2. full capture: per-kernel duration, traffic, IPC, stall top-5
rep = os.path.join(G, "prof_full.ncu-rep")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
h = rr[0]
unit_row = dict(zip(h, rr[1]))
SCALE = {"": 1.0, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6, "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6}
out = {}
txt = [f"# ncu --set full --clock-control none, tools/prof_gs.py 4096 64 2 (64 targets of 4096^2, the bench batch)"]
for r in rr[2:]:
    d = dict(zip(h, r))
    name = d["Kernel Name"].split("(")[0].replace("void ", "")
    if name in out:
        continue
    def f(k):
        if d.get(k, "") in ("", None):
            return None
        return float(d[k].replace(",", "")) * SCALE.get(unit_row.get(k, ""), 1.0)
    rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
    units = {"dram__bytes_read.sum": d.get("dram__bytes_read.sum"), }
    stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""): f(k)
              for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
    top = sorted(((v, k) for k, v in stalls.items() if v), reverse=True)[:5]
    out[name] = {"duration_us": f("gpu__time_duration.sum"), "dram_read_bytes": rd, "dram_write_bytes": wr,
                 "ipc": f("sm__inst_executed.avg.per_cycle_active"),
                 "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                 "warps_per_sm": f("sm__warps_active.avg.per_cycle_active"),
                 "registers": f("launch__registers_per_thread"),
                 "dram_throughput_pct": f("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                 "fma_pipe_pct": f("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                 "top_stalls": [[k, round(v, 2)] for v, k in top]}
    txt.append(f"{name}: {json.dumps(out[name])}")
open(os.path.join(P, f"{tag}_ncu_full_summary.txt"), "w").write("\n".join(txt) + "\n")
print("\n".join(txt))
# traffic per launch for bench.py (dram bytes of one launch of the 64-target batch)
traffic = {}
# the fused GS passes: the persistent row pass of the K-1 non-final iterations
# (k_row_persist<N, QK_FULL, no Q, no levels>, else k_row<N, ROW_FUSED, ...>) and
# k_col<N, C, COL_GS_FAST (3), ...>
for name, key in (("k_row_persist<4096, 2, 0, 0>", "gs_row"), ("k_row<4096, 0,", "gs_row"),
                  ("k_col<4096, 2, 3,", "gs_col")):
    if key in traffic:
        continue
    for k, v in out.items():
        if k.startswith("hg::" + name) or k.startswith(name):
            if v["dram_read_bytes"] is not None:
                traffic[key] = v["dram_read_bytes"] + v["dram_write_bytes"]
                break
traffic["source"] = (f"profiles/{tag}_ncu_full_summary.txt: ncu --set full of tools/prof_gs.py 4096 64 2 (64 targets), "
                     "dram__bytes_read.sum + dram__bytes_write.sum per launch; algorithmic 17.18 GB (row) / 21.47 GB (col)")
json.dump(traffic, open(os.path.join(P, "traffic.json"), "w"), indent=1)
print(traffic)
