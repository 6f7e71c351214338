"""Summarise a gpu_check.sh run's ncu output into tracked files under profiles/.

    python scripts/ncu_summary.py gpurun_out/<tag> <prefix>

Writes
  profiles/<prefix>_launches.txt  per-kernel device time and share of the step
                                  (ncu launch list: cold-cache, serialised —
                                  compare shares, not absolutes)
  profiles/<prefix>_full.txt      key `ncu --set full` metrics per captured launch
  profiles/ncu_traffic.json       dram bytes per launch per kernel (merged);
                                  bench.py reports it as roofline.traffic
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def short(name: str) -> str:
    n = name.split("(")[0]
    n = n.replace("void ", "")
    tmpl = ""
    if "<" in n:
        n, tmpl = n.split("<", 1)
        tmpl = "<" + tmpl
    return n.split("::")[-1] + tmpl


def to_us(v: float, unit: str) -> float:
    return {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0,
            "ms": 1e3, "msecond": 1e3}.get(unit, 1.0) * v


def launches(src: str, steps: int):
    rows = list(csv.reader(open(src)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi or not r[vi]:
            continue
        v = to_us(float(r[vi].replace(",", "")), r[ui])
        k = short(r[ki])
        tot[k] += v
        cnt[k] += 1
    T = sum(tot.values())
    out = [f"# ncu launch list ({src}); {sum(cnt.values())} launches, "
           f"{T:.1f} us total; per step = total / {steps} captured steps",
           f"{'kernel':34s} {'launches':>8s} {'us/launch':>10s} {'us total':>10s} {'share':>7s}"]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        out.append(f"{k:34s} {cnt[k]:8d} {v / cnt[k]:10.1f} {v:10.1f} {v / T * 100:6.1f}%")
    return "\n".join(out) + "\n"


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__t_bytes.sum", "launch__grid_size", "launch__block_size",
           "launch__registers_per_thread", "launch__shared_mem_per_block_dynamic",
           "launch__shared_mem_per_block_static",
           "sm__warps_active.avg.pct_of_peak_sustained_active",
           "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
           "smsp__average_warp_latency_issue_stalled_long_scoreboard",
           "smsp__issue_active.avg.pct_of_peak_sustained_active"]

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def full(rep: str):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    lines = [f"# ncu --set full ({rep})"]
    traffic = {}
    for r in rows[2:]:
        k = short(r[h.index("Kernel Name")])
        lines.append(f"## {k}")
        vals = {}
        for m in METRICS:
            if m in h:
                i = h.index(m)
                lines.append(f"  {m:60s} {r[i]:>14s} {units[i]}")
                vals[m] = (r[i], units[i])
        rb = float(vals["dram__bytes_read.sum"][0].replace(",", "")) * SCALE.get(
            vals["dram__bytes_read.sum"][1], 1)
        wb = float(vals["dram__bytes_write.sum"][0].replace(",", "")) * SCALE.get(
            vals["dram__bytes_write.sum"][1], 1)
        traffic.setdefault(k.split("<")[0], []).append(rb + wb)
    return "\n".join(lines) + "\n", {k: sum(v) / len(v) for k, v in traffic.items()}


def main():
    src, prefix = sys.argv[1], sys.argv[2]
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    prof = os.path.join(ROOT, "profiles")
    os.makedirs(prof, exist_ok=True)
    if os.path.exists(os.path.join(src, "launches.csv")):
        open(os.path.join(prof, f"{prefix}_launches.txt"), "w").write(
            launches(os.path.join(src, "launches.csv"), steps))
    rep = os.path.join(src, "prof.ncu-rep")
    if os.path.exists(rep):
        txt, tr = full(rep)
        open(os.path.join(prof, f"{prefix}_full.txt"), "w").write(txt)
        tj = os.path.join(prof, "ncu_traffic.json")
        cur = json.load(open(tj)) if os.path.exists(tj) else {}
        for k, v in tr.items():
            cur[k] = {"dram_bytes_per_launch": v, "source": f"{prefix}_full.txt"}
        json.dump(cur, open(tj, "w"), indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
