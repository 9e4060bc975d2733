#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) and
an ncu --set full report (.ncu-rep) into profiles/<tag>.json, and update
profiles/ncu_raster_traffic.json (DRAM bytes per raster launch, read by
bench.py for the roofline "traffic" field).

usage: scripts/ncu_summary.py TAG CONFIG LAUNCHES.csv REPORT.ncu-rep
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
           "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "smsp__inst_executed.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
           "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__t_sectors_srcunit_tex_op_atom.sum", "lts__t_sectors_srcunit_tex_op_red.sum",
           "smsp__pcsamp_warps_issue_stalled_short_scoreboard", "smsp__pcsamp_warps_issue_stalled_wait",
           "smsp__pcsamp_warps_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_barrier",
           "smsp__pcsamp_warps_issue_stalled_math_pipe_throttle", "smsp__pcsamp_warps_issue_stalled_not_selected",
           "smsp__pcsamp_warps_issue_stalled_selected", "smsp__pcsamp_warps_issue_stalled_mio_throttle",
           "smsp__pcsamp_warps_issue_stalled_lg_throttle"]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def short(name):
    name = name.replace("void ", "")
    name = re.sub(r"\(.*$", "", name)
    return name.replace("smoe::", "")


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) > vi:
            agg.setdefault(short(r[ki]), []).append(float(r[vi].replace(",", "")) / 1e3)
    return {k: {"n": len(v), "mean_us": sum(v) / len(v), "min_us": min(v), "max_us": max(v)} for k, v in agg.items()}


def full(rep):
    txt = subprocess.check_output(["ncu", "-i", rep, "--page", "raw", "--csv"], stderr=subprocess.DEVNULL).decode()
    rows = list(csv.reader(io.StringIO(txt)))
    H, U = rows[0], rows[1]
    out = {}
    for r in rows[2:]:
        name = short(r[H.index("Kernel Name")])
        d = {}
        for m in METRICS:
            if m in H:
                v = r[H.index(m)].replace(",", "")
                u = U[H.index(m)]
                try:
                    fv = float(v)
                except ValueError:
                    continue
                if u in SCALE:
                    d[m + " [byte]"] = fv * SCALE[u]
                else:
                    d[m + (f" [{u}]" if u else "")] = fv
        out.setdefault(name, d)
    return out


def main():
    tag, cfg, lpath, rep = sys.argv[1:5]
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = {"tag": tag, "config": cfg, "launch_list": launches(lpath), "full_capture": full(rep)}
    # share of the step from the cold, serialised launch list
    ll = res["launch_list"]
    ours = {k: v for k, v in ll.items() if k.startswith("k_")}
    tot = sum(v["mean_us"] * v["n"] for v in ours.values())
    res["share_of_library_time"] = {k: v["mean_us"] * v["n"] / tot for k, v in ours.items()}
    pdir = os.environ.get("SMOE_PROFILES_DIR", os.path.join(root, "profiles"))
    os.makedirs(pdir, exist_ok=True)
    json.dump(res, open(os.path.join(pdir, f"{tag}.json"), "w"), indent=1)
    tpath = os.path.join(pdir, "ncu_raster_traffic.json")
    if not os.path.exists(tpath) and os.path.exists(os.path.join(root, "profiles", "ncu_raster_traffic.json")):
        import shutil
        shutil.copy(os.path.join(root, "profiles", "ncu_raster_traffic.json"), tpath)
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for k, d in res["full_capture"].items():
        if k.startswith("k_raster") and k.endswith(", 1, 1>") or (k.startswith("k_raster") and ", 1," in k):
            b = d.get("dram__bytes_read.sum [byte]", 0.0) + d.get("dram__bytes_write.sum [byte]", 0.0)
            traffic[cfg] = {"kernel": k, "dram_bytes_per_launch": b, "source": f"profiles/{tag}.json"}
            break
    json.dump(traffic, open(tpath, "w"), indent=1)
    print(json.dumps(res["launch_list"], indent=1))
    print(json.dumps(res["share_of_library_time"], indent=1))


if __name__ == "__main__":
    main()
