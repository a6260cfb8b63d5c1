"""Summarise gpurun_out/traffic_<cfg>.csv (ncu metrics of two eager V(1,1) cycles) into per-kernel
DRAM bytes and durations for the second cycle; writes profiles/r2_ncu_traffic.json and .md."""
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from workloads import get_config

out, md = {}, ["# ncu DRAM traffic per kernel, second eager V(1,1) cycle (round 2)", "",
               "`scripts/gpu_traffic.sh` (ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
               "dram__bytes_write.sum; cold-cache serialised launches, so compare shares/bytes, not absolute times).", ""]
for cfg in ("c1", "c2", "c3", "c4", "c5"):
    fn = os.path.join(ROOT, "gpurun_out", "traffic_%s.csv" % cfg)
    if not os.path.exists(fn):
        continue
    rows = [r for r in csv.reader(l for l in open(fn) if l.startswith('"'))]
    hdr = rows[0]
    ik, im, iv, iid = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("ID")
    launches = {}
    for r in rows[1:]:
        name = r[ik]
        if "pmg::" not in name and "unnamed>::" not in name:
            continue
        d = launches.setdefault(int(r[iid]), {"name": name})
        val = float(r[iv].replace(",", ""))
        unit = r[hdr.index("Metric Unit")]
        if r[im] == "gpu__time_duration.sum":                    # -> microseconds
            val *= {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(unit, 1.0)
        elif r[im].startswith("dram__bytes"):                    # -> bytes
            val *= {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1.0)
        d[r[im]] = val
    ids = sorted(launches)
    half = ids[len(ids) // 2:]                      # second cycle
    agg = {}
    for i in half:
        L = launches[i]
        m = re.search(r"(k_\w+)", L["name"])
        short = m.group(1) if m else L["name"][:40]
        j = m.end() if m else 0
        if j < len(L["name"]) and L["name"][j] == "<":          # template arguments up to the matching '>'
            depth, k = 0, j
            while k < len(L["name"]):
                depth += {"<": 1, ">": -1}.get(L["name"][k], 0)
                k += 1
                if depth == 0:
                    break
            short += re.sub(r"\((int|bool)\)", "", L["name"][j:k])
        a = agg.setdefault(short, {"launches": 0, "us": 0.0, "read": 0.0, "write": 0.0})
        a["launches"] += 1
        a["us"] += L.get("gpu__time_duration.sum", 0.0)
        a["read"] += L.get("dram__bytes_read.sum", 0.0)
        a["write"] += L.get("dram__bytes_write.sum", 0.0)
    c = get_config(cfg)
    tot_us = sum(a["us"] for a in agg.values())
    out[cfg] = {"dofs": c.ndofs, "kernels": agg, "cycle_us": tot_us,
                "cycle_dram_bytes": sum(a["read"] + a["write"] for a in agg.values())}
    md += ["## %s (%d DOF; cycle %.1f us, DRAM %.1f MB)" % (cfg, c.ndofs, tot_us, out[cfg]["cycle_dram_bytes"] / 1e6), "",
           "| kernel | launches | us | share | DRAM read MB | DRAM write MB | B/DOF |", "|---|---|---|---|---|---|---|"]
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
        md.append("| %s | %d | %.1f | %.1f%% | %.1f | %.1f | %.1f |" % (
            k, a["launches"], a["us"], 100 * a["us"] / tot_us, a["read"] / 1e6, a["write"] / 1e6,
            (a["read"] + a["write"]) / c.ndofs))
    md.append("")
json.dump(out, open(os.path.join(ROOT, "profiles", "r2_ncu_traffic.json"), "w"), indent=1)
open(os.path.join(ROOT, "profiles", "r2_ncu_traffic.md"), "w").write("\n".join(md) + "\n")
print("\n".join(md))
