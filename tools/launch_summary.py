"""Dev tool: summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into per-kernel
launches / total / average / share, and per bench.py kernel class.  ncu times are cold-cache and
serialised: compare SHARES with bench.py's live kernel classes, not absolute times.

usage: python tools/launch_summary.py gpurun_out/launches.csv "<command line>" > profiles/rNN_launches_summary.csv
"""
import csv
import re
import sys
from collections import defaultdict

CLASSES = [  # (regex on the demangled name, bench.py class)
    (r"k_b_sweepc?<0", "batched ic fwd sweep (k_b_sweepc<false>)"),
    (r"k_b_sweepc?<1|k_b_rho", "batched ic bwd sweep (k_b_sweepc<true> + k_b_rho)"),
    (r"k_b_spmv_pq|k_b_residual", "batched spmv (k_b_spmv_pq)"),
    (r"k_b_tallt", "batched W^T r (k_b_tallt)"),
    (r"k_b_", "batched vector ops"),
    (r"k_sweep<0", "ic fwd sweep (k_sweep<false>)"),
    (r"k_sweep<1", "ic bwd sweep (k_sweep<true>)"),
    (r"k_spmv_pq|k_residual|k_spmv<", "spmv (k_spmv_pq)"),
    (r"k_tallt", "W^T r (k_tallt)"),
]


def cls_of(name):
    for rx, c in CLASSES:
        if re.search(rx, name):
            return c
    return "other (setup / recycling / vector ops)"


def main():
    path, cmd = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
    rows = []
    with open(path) as f:
        lines = [ln for ln in f if ln.startswith('"')]
    rd = csv.DictReader(lines)
    for r in rd:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        unit = r.get("Metric Unit", "ns")
        v = float(r["Metric Value"].replace(",", ""))
        us = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
        rows.append((r["Kernel Name"], us))
    per_k = defaultdict(lambda: [0, 0.0])
    per_c = defaultdict(lambda: [0, 0.0])
    for name, us in rows:
        short = re.sub(r"\(.*", "", name.replace("void ", "").replace("rcg::", ""))
        tmpl = re.search(r"<[^>]*>", name)
        key = short + (tmpl.group(0) if tmpl and "<" not in short else "")
        per_k[key][0] += 1
        per_k[key][1] += us
        c = cls_of(name)
        per_c[c][0] += 1
        per_c[c][1] += us
    tot = sum(us for _, us in rows)
    print(f"# {cmd}")
    print("# cold-cache, serialised launches (ncu): compare SHARES with bench.py kernel classes")
    print("kind,name,launches,total_us,avg_us,share")
    for c, (k, us) in sorted(per_c.items(), key=lambda x: -x[1][1]):
        print(f"class,{c},{k},{us:.1f},{us / k:.2f},{us / tot:.4f}")
    for name, (k, us) in sorted(per_k.items(), key=lambda x: -x[1][1])[:25]:
        print(f"kernel,{name},{k},{us:.1f},{us / k:.2f},{us / tot:.4f}")


if __name__ == "__main__":
    main()
