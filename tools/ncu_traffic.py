"""DRAM traffic per launch of each bench kernel class from an ncu launch list.

    python tools/ncu_traffic.py LAUNCHES.csv [OUT.json [WINDOW [ALGO.json]]]

ALGO.json (bench.py under CORTEX_NCU_TIMED=1) holds the algorithmic bytes of the same
launches: each class then also gets dram_per_algorithmic_byte, the re-read factor.

The CSV is `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
--csv --log-file ...` of a bench.py run. Kernel names map to the classes bench.py times
with CUDA events (gemm / attn_decode / attn_prefill); the JSON (profiles/traffic.json)
is what bench.py reports as roofline.traffic for the dominant class, next to the
algorithmic bytes per launch it measures live.
"""

from __future__ import annotations

import collections
import csv
import json
import sys

CLASSES = {
    "gemm": ("gemm_bf16",),
    "attn_decode": ("paged_decode", "cascade_prefix", "decode_combine", "fmha_tc_kernel",
                    "fmha2_tc_kernel"),
    "attn_prefill": ("fmha_tc_kernel", "fmha2_tc_kernel", "paged_prefill"),
    "attn_decode_ctx": ("paged_decode",),
}


def per_kernel(path: str) -> dict:
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ii, ki, mi, vi, ui = (h.index(c) for c in ("ID", "Kernel Name", "Metric Name",
                                                 "Metric Value", "Metric Unit"))
    launches: dict = collections.defaultdict(dict)
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
        v = float(r[vi].replace(",", ""))
        unit = r[ui]
        if r[mi] == "gpu__time_duration.sum":
            v = {"ns": v / 1e3, "nsecond": v / 1e3, "us": v, "usecond": v, "ms": v * 1e3}.get(unit, v)
        else:
            v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6,
                  "GB": 1e9}.get(unit, 1)
        launches[r[ii]]["name"] = name
        launches[r[ii]][r[mi]] = v
    return launches


def summarize(path: str, window: str | None = None) -> dict:
    launches = per_kernel(path)
    out = {"source": path, "window": window, "classes": {}}
    for cls, keys in CLASSES.items():
        sel = [d for d in launches.values() if any(k in d["name"] for k in keys)]
        if not sel:
            continue
        n = len(sel)
        rd = sum(d.get("dram__bytes_read.sum", 0.0) for d in sel)
        wr = sum(d.get("dram__bytes_write.sum", 0.0) for d in sel)
        us = sum(d.get("gpu__time_duration.sum", 0.0) for d in sel)
        out["classes"][cls] = {"launches": n, "dram_bytes_per_launch": (rd + wr) / n,
                               "dram_read_per_launch": rd / n, "dram_write_per_launch": wr / n,
                               "us_per_launch": us / n}
    return out


if __name__ == "__main__":
    res = summarize(sys.argv[1], sys.argv[3] if len(sys.argv) > 3 else None)
    if len(sys.argv) > 4:
        algo = json.load(open(sys.argv[4]))
        for cls, v in res["classes"].items():
            a = algo.get(cls)
            if a and a["launches"] == v["launches"]:  # the same launches
                v["algorithmic_bytes_per_launch"] = a["bytes"] / a["launches"]
                v["dram_per_algorithmic_byte"] = v["dram_bytes_per_launch"] / (
                    a["bytes"] / a["launches"])
    print(json.dumps(res, indent=1))
    if len(sys.argv) > 2:
        with open(sys.argv[2], "w") as f:
            json.dump(res, f, indent=1)
