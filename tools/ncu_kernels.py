"""Dev tool: per-kernel summary of an `ncu --set full` capture exported with
`ncu -i REP --page raw --csv` (duration, DRAM bytes read / written, achieved DRAM GB/s, L2
throughput %, registers, warps active), and the per-class DRAM bytes bench.py reports as
`roofline.traffic` (profiles/ncu_traffic.json, keyed by workload).

  python tools/ncu_kernels.py gpurun_out/prof_c3b_raw.csv gpurun_out/prof_c3s_raw.csv \
      --workload c3_q1_27pt_256 --rt 24 --note "..." > profiles/r2_ncu_c3_kernels.csv
"""
import argparse
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
from launch_summary import cls_of  # noqa: E402

COLS = {"dur": "gpu__time_duration.sum", "rd": "dram__bytes_read.sum", "wr": "dram__bytes_write.sum",
        "l2": "lts__t_sectors_op_read.sum", "regs": "launch__registers_per_thread",
        "warps": "sm__warps_active.avg.pct_of_peak_sustained_active"}


def rows(path):
    with open(path) as f:
        rd = list(csv.reader(f))
    hdr = next(i for i, r in enumerate(rd) if "Kernel Name" in r)
    names = rd[hdr]
    units = rd[hdr + 1]
    out = []
    for r in rd[hdr + 2:]:
        if len(r) != len(names):
            continue
        d = dict(zip(names, r))
        u = dict(zip(names, units))
        out.append((d, u))
    return out


def num(d, u, key, scale_to):
    v = d.get(key, "")
    if v in ("", "n/a"):
        return None
    v = float(v.replace(",", ""))
    unit = u.get(key, "")
    mult = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6,
            "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(unit, 1.0)
    return v * mult


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("csvs", nargs="+")
    ap.add_argument("--workload", required=True)
    ap.add_argument("--rt", type=int, default=0, help="right-hand sides per batched launch in the capture")
    ap.add_argument("--note", default="")
    ap.add_argument("--update-traffic", action="store_true", help="write profiles/ncu_traffic.json[workload]")
    args = ap.parse_args()
    per_class = {}
    print(f"# ncu --set full --clock-control none (cold cache, serialised launches): {args.note}")
    print("kernel,class,duration_us,dram_read_B,dram_write_B,dram_GBps,regs,warps_active_pct")
    for path in args.csvs:
        for d, u in rows(path):
            name = d.get("Kernel Name", "?")
            short = re.sub(r"\(.*", "", name).replace("void rcg::", "").replace("rcg::", "")
            dur = num(d, u, COLS["dur"], "us")
            rd = num(d, u, COLS["rd"], "B") or 0.0
            wr = num(d, u, COLS["wr"], "B") or 0.0
            gbps = (rd + wr) / (dur * 1e-6) / 1e9 if dur else 0.0
            c = cls_of(short)
            print(f'"{short}",{c},{dur:.1f},{int(rd)},{int(wr)},{gbps:.1f},{d.get(COLS["regs"], "")},'
                  f'{d.get(COLS["warps"], "")}')
            per_class.setdefault(c, {}).setdefault(re.sub(r"<.*", "", short), []).append(rd + wr)
    if args.update_traffic:
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        t = json.load(open(tp)) if os.path.exists(tp) else {}
        entry = {"_source": args.note}
        for c, by_name in per_class.items():
            # one bench.py class launch: the backward sweep class is the sweep AND its k_b_rho
            # (one KTimer), every other class one kernel per launch (mean over its launches)
            means = {k: sum(v) / len(v) for k, v in by_name.items()}
            b = int(sum(means.values())) if "bwd" in c else int(sum(sum(v) for v in by_name.values()) /
                                                               sum(len(v) for v in by_name.values()))
            entry[c] = {"dram_bytes": b, "rhs_per_launch": args.rt, "algorithmic_bytes": None} if c.startswith("batched") else b
        t[args.workload] = entry
        json.dump(t, open(tp, "w"), indent=1)


if __name__ == "__main__":
    main()
