"""Dev tool: merge the parity records the GPU tests wrote (tests/conftest.py `parity_log` ->
gpurun_out/parity/*.jsonl: achieved difference and bar per check) into one committed file.

  python tools/parity_summary.py > profiles/parity_r2.json
"""
import glob
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main():
    recs = {}
    for path in sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "parity", "*.jsonl"))):
        with open(path) as f:
            for line in f:
                line = line.strip()
                if not line:
                    continue
                r = json.loads(line)
                recs.setdefault(r.pop("test"), []).append(r)
    out = {"_note": "achieved value and bar of every logged parity check of one `pytest -m gpu` run on a B200 "
                    "(tests/conftest.py parity_log); one list per check, one entry per call",
           "checks": {k: recs[k] for k in sorted(recs)}}
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
