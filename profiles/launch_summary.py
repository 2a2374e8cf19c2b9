"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list.

    python profiles/launch_summary.py gpurun_out/launches.csv [--top 30]
"""
import collections
import csv
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
         "s": 1e6, "second": 1e6}


def summarise(path, top=30):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        us = float(r[vi].replace(",", "")) * SCALE[r[ui]]
        a = agg.setdefault(r[ki][:100], [0, 0.0])
        a[0] += 1
        a[1] += us
    tot = sum(v[1] for v in agg.values())
    out = [f"{'ms':>10} {'share':>6} {'launches':>8}  kernel"]
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
        out.append(f"{v[1] / 1e3:10.3f} {100 * v[1] / tot:5.1f}% {v[0]:8d}  {k}")
    out.append(f"total {tot / 1e3:.3f} ms over {sum(v[0] for v in agg.values())} launches")
    return "\n".join(out)


if __name__ == "__main__":
    print(summarise(sys.argv[1], int(sys.argv[3]) if len(sys.argv) > 3 else 30))
