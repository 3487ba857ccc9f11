"""Summarise an `ncu --metrics gpu__time_duration.sum --csv` launch list: per-kernel launches, total ms, share.

    python tools/launch_summary.py gpurun_out/launches_c2.csv "header line" > profiles/r01_launches_c2_summary.txt
"""
import collections
import csv
import sys

SCALE = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}


def main(path, header):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, mi, vi, ui = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) > vi and r[mi] == "gpu__time_duration.sum":
            name = r[ki].split("(")[0]
            tot[name] += SCALE[r[ui]] * float(r[vi].replace(",", ""))
            cnt[name] += 1
    T = sum(tot.values())
    print(header)
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        print(f"{k:60s} launches={cnt[k]:4d} total={v:9.3f} ms share={v / T:.3f}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "")
