"""One-line-per-kernel summaries of ncu --set full reports (duration, DRAM
bytes, pipe / L1 / issue utilisation, top warp stalls).
  python tools/ncu_summary.py report.ncu-rep [...]"""
import csv
import io
import re
import subprocess
import sys

KEYS = {"gpu__time_duration.sum": "duration_us_ns", "dram__bytes_read.sum": "dram_read",
        "dram__bytes_write.sum": "dram_write", "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
        "l1tex__throughput.avg.pct_of_peak_sustained_active": "l1tex_pct",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
        "sm__warps_active.avg.per_cycle_active": "warps_per_sm", "launch__registers_per_thread": "registers",
        "smsp__inst_executed.sum": "warp_instructions"}


def main():
    for rep in sys.argv[1:]:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(out)))
        hdr, units, data = rows[0], rows[1], rows[2:]
        kn = hdr.index("Kernel Name")
        print(f"# {rep}")
        for d in data:
            r = {}
            for k, name in KEYS.items():
                if k in hdr:
                    v = d[hdr.index(k)].replace(",", "")
                    u = units[hdr.index(k)]
                    try:
                        v = float(v)
                    except ValueError:
                        continue
                    if k == "gpu__time_duration.sum":
                        name, v = "duration_us", v / 1e3 if u == "ns" else (v * 1e3 if u == "ms" else v)
                    if k.startswith("dram__bytes"):
                        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                        v = v * scale
                    r[name] = round(v, 3)
            st = {}
            for i, h in enumerate(hdr):
                m = re.match(r"smsp__pcsamp_warps_issue_stalled_(\w+)$", h)
                if m and not h.endswith("not_issued") and d[i]:
                    st[m.group(1)] = float(d[i])
            tot = sum(st.values()) or 1.0
            r["top_stalls_pct"] = [(k, round(100 * v / tot, 1)) for k, v in sorted(st.items(), key=lambda kv: -kv[1])[:6]]
            print(f"{d[kn][:70]}: {r}")


if __name__ == "__main__":
    main()
