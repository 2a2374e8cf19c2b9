"""Stall-reason breakdown of an ncu --set full report, per source-line range.

    python profiles/ncu_stalls.py x.ncu-rep file.cu "{'phase': (lo, hi), ...}"
"""
import csv
import io
import subprocess
import sys


def main(rep, fname, ranges):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur, hdr, agg = None, None, {}
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r and r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr) or r[2] != "-":
            continue
        try:
            ln = int(r[0])
        except ValueError:
            continue
        name = "other"
        if cur == fname:
            for nm, (a, b) in ranges.items():
                if a <= ln <= b:
                    name = nm
                    break
        d = agg.setdefault(name, {})
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    d[h[6:]] = d.get(h[6:], 0) + float(r[i])
                except ValueError:
                    pass
    tot = sum(sum(d.values()) for d in agg.values()) or 1
    for nm, d in sorted(agg.items(), key=lambda kv: -sum(kv[1].values())):
        s = sum(d.values())
        top = sorted(d.items(), key=lambda kv: -kv[1])[:6]
        print(f"{nm:12s} {100 * s / tot:5.1f}%  " + "  ".join(f"{k}={100 * v / tot:.1f}" for k, v in top if v))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], eval(sys.argv[3]))
