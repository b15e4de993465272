"""Summarise ncu output into profiles/ (tracked).

  python tools/ncu_summarize.py launches <launches.csv> <out.json>
      per-kernel device-time shares from an `ncu --metrics gpu__time_duration.sum` list
  python tools/ncu_summarize.py report <file.ncu-rep> <out.json> [workload group]
      key counters of a `--set full` capture (duration, DRAM bytes, occupancy,
      issue activity, stall breakdown); with workload/group also records
      dram_bytes_per_launch in profiles/ncu_summary.json for bench.py's roofline
"""
import collections
import csv
import io
import json
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name):
    m = re.search(r"::(\w+?)(?:<|\()", name)
    return m.group(1) if m else name[:60]


def launches(path, out):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows[1:]:
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
                 "nsecond": 1e-3}.get(r[ui], 1.0)
        tot[short(r[ki])] += v * scale
        cnt[short(r[ki])] += 1
    total = sum(tot.values())
    res = {"source": os.path.basename(path), "launches": sum(cnt.values()),
           "total_us": round(total, 1),
           "kernels": {k: {"us": round(v, 1), "share": round(v / total, 4), "launches": cnt[k]}
                       for k, v in tot.most_common()}}
    json.dump(res, open(out, "w"), indent=1)
    return res


def report(path, out, workload=None, group=None):
    # base units: every row in ns / bytes (auto units change per row)
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr = rows[0]
    res = {"source": os.path.basename(path), "launches": []}
    for r in rows[2:]:
        d = dict(zip(hdr, r))

        def f(k):
            try:
                return float(d[k].replace(",", ""))
            except (KeyError, ValueError):
                return None
        stalls = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): f(k) for k in hdr
                  if k.startswith("smsp__pcsamp_warps_issue_stalled_") and
                  not k.endswith("not_issued") and f(k)}
        st = sum(stalls.values()) or 1.0
        rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
        mult = 1
        launch = {
            "kernel": short(d.get("Kernel Name", "")), "grid": d.get("Grid Size"),
            "block": d.get("Block Size"),
            "duration_ms": f("gpu__time_duration.sum") / 1e6,
            "dram_bytes": (rd + wr) * mult if rd is not None and wr is not None else None,
            "warps_active_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
            "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "fp64_pipe_pct": f("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"),
            "registers": f("launch__registers_per_thread"),
            "stall_share": {k: round(v / st, 3) for k, v in sorted(stalls.items(),
                                                                   key=lambda x: -x[1])[:8]},
        }
        res["launches"].append(launch)
    json.dump(res, open(out, "w"), indent=1)
    if workload and group and res["launches"]:
        sp = os.path.join(ROOT, "profiles", "ncu_summary.json")
        summ = json.load(open(sp)) if os.path.exists(sp) else {}
        b = [l["dram_bytes"] for l in res["launches"] if l["dram_bytes"] is not None]
        summ.setdefault(workload, {})[group] = {
            "dram_bytes_per_launch": sum(b) / len(b) if b else None,
            "duration_ms": res["launches"][0]["duration_ms"], "source": os.path.basename(path)}
        json.dump(summ, open(sp, "w"), indent=1)
    return res


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(json.dumps(launches(sys.argv[2], sys.argv[3]))[:2000])
    else:
        print(json.dumps(report(*sys.argv[2:]))[:3000])
