"""Dev: per-kernel SASS instruction counts of the product library (cuobjdump -sass): the bulk
copies (UBLKCP = cp.async.bulk), mbarrier ops (SYNCS), 256-bit relaxed / plain global accesses
(LDG/STG ...ENL2.256), FP64 (DADD/DMUL/DFMA), shuffles, spills (LDL/STL).
  python tools/sass_summary.py > profiles/sass_summary_r2.txt"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
so = os.path.join(ROOT, "paper_2203_08498_b200", "librcg_b200.so")
out = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
KEYS = [("UBLKCP", r"\bUBLKCP"), ("SYNCS", r"\bSYNCS"), ("LDG.256", r"\bLDG\.E\.[A-Z0-9.]*ENL2\.256"),
        ("STG.256", r"\bSTG\.E\.[A-Z0-9.]*ENL2\.256"), ("LDG", r"\bLDG\b"), ("STG", r"\bSTG\b"),
        ("LDS", r"\bLDS\b"), ("DFMA", r"\bDFMA\b"), ("DADD", r"\bDADD\b"), ("DMUL", r"\bDMUL\b"),
        ("SHFL", r"\bSHFL\b"), ("LDL/STL (spill)", r"\b(LDL|STL)\b"), ("tcgen05/UTC", r"\bUTC")]
cur, counts = None, collections.OrderedDict()
for line in out.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        counts[cur] = collections.Counter()
        continue
    if cur is None:
        continue
    for k, rx in KEYS:
        if re.search(rx, line):
            counts[cur][k] += 1
demangled = {}
try:
    names = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
    demangled = dict(zip(counts, names))
except OSError:
    pass
hot = re.compile(r"k_sweep|k_b_sweepc|k_spmv|k_b_spmv|k_b_tallt|k_b_deflate|k_b_pupdate|k_b_xr|k_b_rho|k_tallt|k_pupdate|k_xr|"
                 r"k_level|k_b_level|k_ic_factor|k_mgs|k_gram|k_spmm|k_harvest|k_b_fin|k_d_")
print("# SASS summary of librcg_b200.so (sm_100a), hot-path kernels; counts of instructions in the kernel body")
print("kernel," + ",".join(k for k, _ in KEYS))
for f, c in counts.items():
    name = demangled.get(f, f)
    if not hot.search(name):
        continue
    print(f'"{name[:110]}",' + ",".join(str(c[k]) for k, _ in KEYS))
tot = collections.Counter()
for c in counts.values():
    tot.update(c)
print("TOTAL (all kernels)," + ",".join(str(tot[k]) for k, _ in KEYS))
