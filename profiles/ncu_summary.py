"""Summarise one ncu --set full capture of a hot-path kernel into the JSON the
bench reads (roofline.traffic, roofline.issue_roof), tagged with the hash of
the CUDA sources it was built from.

    python profiles/ncu_summary.py gpurun_out/x.ncu-rep <config> <kernel-tag> [launch-index]
      -> profiles/<config>_<kernel-tag>_ncu.json
"""
import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import bench  # noqa: E402

KEYS = {
    "gpu__time_duration.sum": "duration_us",
    "smsp__inst_executed.sum": "inst_executed",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_slots_busy_pct",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "smsp__cycles_active.avg": "cycles_active",
    "sm__cycles_elapsed.avg.per_second": "sm_hz",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__registers_per_thread": "registers",
}
UNITS = {"dram_read": {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9},
         "dram_write": {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9},
         "duration_us": {"ns": 1e-3, "us": 1.0, "ms": 1e3, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3},
         "sm_hz": {"hz": 1.0, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "cycle/second": 1.0, "cycle/nsecond": 1e9}}


def main(rep, config, tag, idx=0):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    r = data[int(idx)]
    d = {"kernel": r[hdr.index("Kernel Name")][:120], "report": os.path.basename(rep)}
    for k, name in KEYS.items():
        if k in hdr:
            i = hdr.index(k)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            v *= UNITS.get(name, {}).get(units[i], 1.0)
            d[name] = v
    d["dram_bytes_per_launch"] = d.get("dram_read", 0.0) + d.get("dram_write", 0.0)
    if "sm_hz" in d:
        d["sm_mhz"] = d["sm_hz"] / 1e6
    d["src_sha"] = bench.kernel_source_hash()
    path = os.path.join(HERE, f"{config}_{tag}_ncu.json")
    with open(path, "w") as fh:
        json.dump(d, fh, indent=1)
    print(path, json.dumps(d))


if __name__ == "__main__":
    main(*sys.argv[1:])
