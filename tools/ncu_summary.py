"""Summarise an ncu capture + launch list into profiles/ncu_summary_<tag>.json.

    python tools/ncu_summary.py gpurun_out/prof_r01.ncu-rep gpurun_out/launches_r01.csv r01 \
        [config precision tokens_per_launch]

Per kernel (full-set capture): duration, DRAM read/write bytes, DRAM %, tensor
pipe %, SM clock, registers, achieved occupancy. From the launch list (one
window, serialised, cold cache): per-kernel-class share of the window.
"""

from __future__ import annotations

import collections
import csv
import io
import json
import os
import subprocess
import sys

METRICS = {
    "duration_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read_bytes": ("dram__bytes_read.sum", 1.0),
    "dram_write_bytes": ("dram__bytes_write.sum", 1.0),
    "dram_pct": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "tensor_pipe_pct": ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", 1.0),
    "sm_throughput_pct": ("sm__throughput.avg.pct_of_peak_sustained_elapsed", 1.0),
    "sm_clock_hz": ("sm__cycles_elapsed.avg.per_second", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "grid": ("launch__grid_size", 1.0),
}
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3,
              "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3, "ms": 1e6, "s": 1e9,
              "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9}


def short(name):
    base = name.split("(")[0].replace("void ", "")
    return base.strip()


def full_set(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        k = {"kernel": short(r[hdr.index("Kernel Name")])}
        for key, (metric, mul) in METRICS.items():
            if metric not in hdr:
                continue
            i = hdr.index(metric)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                continue
            v *= UNIT_SCALE.get(units[i], 1.0)
            k[key] = v * mul if key == "duration_ms" else v
        res.append(k)
    return res


def launch_list(path):
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows[h + 1:]:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", "")) * UNIT_SCALE.get(r[ui], 1.0)
        agg[short(r[ki])][0] += 1
        agg[short(r[ki])][1] += v
    tot = sum(v[1] for v in agg.values())
    return {k: {"launches": n, "ms": ns / 1e6, "share": ns / tot}
            for k, (n, ns) in sorted(agg.items(), key=lambda x: -x[1][1])}, tot / 1e6


def main(rep, launches, tag, cfg="2", prec="fp32", tokens=None):
    kernels = full_set(rep)
    shares, total_ms = launch_list(launches)
    gemms = [k for k in kernels if k["kernel"].startswith(("gemm_tc_kernel", "gemm2_tc_kernel"))]
    dom = max(gemms, key=lambda k: k.get("duration_ms", 0)) if gemms else None
    summary = {
        "tag": tag,
        "config": int(cfg), "precision": prec,
        "tokens_per_launch": int(tokens) if tokens else None,
        "how": f"ncu --set full --clock-control none (first layer of 1 window of config-{cfg} records, "
               f"precision {prec}, tools/profile_window.py); launch list: ncu --metrics "
               "gpu__time_duration.sum",
        "window_total_ms_serialised": total_ms,
        "launch_shares": shares,
        "kernels": kernels,
        "dominant_gemm": dom,
        "dram_bytes_per_launch": (dom["dram_read_bytes"] + dom["dram_write_bytes"]) if dom else None,
    }
    # the full-set capture is layer 0 of the window in launch order
    order = ["qkv", "attention", "o_proj", "layernorm", "ffn1", "ffn2"]
    if len(kernels) >= len(order):
        summary["by_class"] = {c: dict(kernels[i], dram_bytes=kernels[i].get("dram_read_bytes", 0)
                                       + kernels[i].get("dram_write_bytes", 0))
                               for i, c in enumerate(order)}
    os.makedirs("profiles", exist_ok=True)
    dst = os.path.join("profiles", f"ncu_summary_{tag}.json")
    with open(dst, "w") as f:
        json.dump(summary, f, indent=1)
    print("wrote", dst)


if __name__ == "__main__":
    main(*sys.argv[1:7])
