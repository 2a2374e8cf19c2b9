"""Top source lines of an ncu report by executed instructions and stall samples.

    python profiles/ncu_source_top.py gpurun_out/x.ncu-rep [N]
"""
import csv
import io
import subprocess
import sys


def main(rep, top=30):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    cur, agg = None, {}
    for r in rows:
        if len(r) >= 2 and r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if len(r) > 8 and r[0] not in ("", "Line No") and r[2] == "-":
            try:
                ie, st = float(r[7]), float(r[4])
            except ValueError:
                continue
            key = (cur, int(r[0]), r[1].strip()[:88])
            a = agg.setdefault(key, [0.0, 0.0])
            a[0] += ie
            a[1] += st
    tot = sum(v[0] for v in agg.values()) or 1
    stt = sum(v[1] for v in agg.values()) or 1
    print(f"total warp-instructions {tot:.4g}, stall samples {stt:.0f}")
    for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{100 * v[0] / tot:5.1f}% instr {100 * v[1] / stt:5.1f}% stall  {k[0]}:{k[1]}  {k[2]}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
