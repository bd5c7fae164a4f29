"""Per-kernel SASS evidence for the hot kernels: opcode counts (TMA / bulk
copies, mbarrier syncs, packed FP32, shared-memory traffic, barriers) from
cuobjdump of the built objects, and the ptxas register / spill lines.
  python tools/sass_summary.py > profiles/r02_sass_summary.txt"""
import collections
import glob
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OBJ = os.path.join(ROOT, "paper_2008_12214_b200", "csrc", "build")
HOT = [  # (object, mangled-name regex, label)
    ("k_row_full.o", r"_ZN2hg13k_row_persistILi4096ELi2ELi0ELi0EE", "k_row_persist<4096, QK_FULL, no Q, no levels>  (GS 4096^2 row pass, K-1 iterations)"),
    ("k_row_full.o", r"_ZN2hg13k_row_persistILi4096ELi2ELi0ELi1EE", "k_row_persist<4096, QK_FULL, no Q, levels>     (last iteration)"),
    ("k_row_full.o", r"_ZN2hg5k_rowILi4096ELi0ELi2ELi1ELi0ELi0EE", "k_row<4096, QK_FULL> (non-persistent, small batches)"),
    ("k_col_gs.o", r"_ZN2hg5k_colILi4096ELi2ELi3ELi1EE", "k_col<4096, C=2, COL_GS_FAST>  (GS 4096^2 column pass)"),
    ("k_col_plain.o", r"_ZN2hg5k_colILi4096ELi2ELi0ELi1EE", "k_col<4096, C=2, COL_PLAIN>    (initial inverse columns)"),
    ("k_row_bin.o", r"_ZN2hg5k_rowILi1024ELi0ELi1ELi1ELi0ELi1EE", "k_row<1024, QK_BINARY, levels>   (OSPR row pass, non-persistent)"),
    ("k_col_ospr.o", r"_ZN2hg5k_colILi1024ELi8ELi2ELi1EE", "k_col<1024, C=8, COL_OSPR>     (OSPR accumulating column pass)"),
    ("capi.o", r"_ZN2hg19k_seed_random_phaseILb1EE", "k_seed_random_phase<fast>      (mt19937_64 + double sincos seed)"),
]
GROUPS = {
    "TMA/bulk": ("UTMALDG", "UTMASTG", "UBLKCP", "UTMAPF", "UBLKPF"),
    "mbarrier": ("SYNCS",),
    "FP32 packed": ("FADD2", "FMUL2", "FFMA2"),
    "FP32 scalar": ("FADD", "FMUL", "FFMA"),
    "FP64": ("DADD", "DMUL", "DFMA"),
    "smem ld/st": ("LDS", "STS"),
    "global ld/st": ("LDG", "STG"),
    "local (spill)": ("LDL", "STL"),
    "barrier": ("BAR",),
    "tensor core": ("UTCHMMA", "UTCQMMA", "UTCIMMA", "HMMA"),
}


def functions(obj):
    out = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    funcs, cur = {}, None
    for line in out.splitlines():
        m = re.match(r"\s+Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = collections.Counter()
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)", line)
        if m and cur:
            funcs[cur][m.group(1)] += 1
    return funcs


def ptxas(obj, mangled):
    log = obj + ".log"
    if not os.path.exists(log):
        return ""
    txt = open(log).read()
    i = txt.find("Function properties for " + mangled)
    if i < 0:
        return ""
    m = re.search(r"(\d+ bytes stack frame, \d+ bytes spill stores, \d+ bytes spill loads).*?(Used \d+ registers)",
                  txt[i:], re.S)
    return f"{m.group(2)}; {m.group(1)}" if m else ""


def main():
    print("# SASS opcode groups (static counts) and ptxas resource use of the hot kernels")
    print("# source: cuobjdump -sass paper_2008_12214_b200/csrc/build/*.o (sm_100a), ptxas -v logs")
    cache = {}
    for obj, rx, label in HOT:
        path = os.path.join(OBJ, obj)
        if not os.path.exists(path):
            continue
        if path not in cache:
            cache[path] = functions(path)
        names = [n for n in cache[path] if re.match(rx, n)]
        if not names:
            print(f"\n{label}: not found")
            continue
        n = names[0]
        c = cache[path]
        print(f"\n{label}\n  {n}")
        print("  total instructions:", sum(c[n].values()))
        for g, ops in GROUPS.items():
            tot = sum(v for k, v in c[n].items() if k in ops)
            if tot:
                parts = ", ".join(f"{k} {c[n][k]}" for k in ops if c[n][k])
                print(f"  {g:14s} {tot:6d}  ({parts})")
        print("  ptxas:", ptxas(path, n))


if __name__ == "__main__":
    main()
