"""Write the round's ncu evidence under profiles/:
  - <tag>_launches.txt : per-kernel share of the step from the launch-list csv
    (ncu --metrics gpu__time_duration.sum --clock-control none pass of bench.py)
  - <tag>_ncu_full.txt : per-kernel DRAM bytes / throughputs / occupancy from a
    --set full capture
  - traffic_cfg<C>.json : dram read+write bytes per launch per bench phase (read by bench.py)
usage: python tools/profile_summary.py <tag> <launches.csv> <full.ncu-rep> <cfg>
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
tag, lcsv, rep, cfg = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4]
out_dir = os.environ.get("PROFILE_OUT") or os.path.join(ROOT, "profiles")
os.makedirs(out_dir, exist_ok=True)

from kernel_phase import phase_of  # noqa: E402

rows = [r for r in csv.reader(open(lcsv)) if len(r) > 5] if lcsv != "-" else [["Metric Name"]]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
agg = collections.OrderedDict()
for r in rows[1:]:
    if r[ix["Metric Name"]] != "gpu__time_duration.sum":
        continue
    nm = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")
    ph = phase_of(nm, r[ix["Grid Size"]])
    v = float(r[ix["Metric Value"]].replace(",", ""))
    a = agg.setdefault(ph, [0, 0.0, nm])
    a[0] += 1
    a[1] += v
tot = sum(v[1] for v in agg.values())
with open(os.devnull, "w") if lcsv == "-" else open(os.path.join(out_dir, f"{tag}_launches.txt"), "w") as f:
    f.write(f"# ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised): {lcsv}\n")
    f.write("# phase  launches  total_us  avg_us  share_of_all_launches  kernel\n")
    for ph, (c, t, nm) in sorted(agg.items(), key=lambda x: -x[1][1]):
        f.write(f"{ph:16s} {c:6d} {t / 1e3:10.1f} {t / c / 1e3:8.2f} {t / tot:7.3f}  {nm}\n")

if rep == "-":          # launch list only (no --set full capture this time)
    print(open(os.path.join(out_dir, f"{tag}_launches.txt")).read())
    sys.exit(0)
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M)],
                     capture_output=True, text=True).stdout
r = list(csv.reader(raw.splitlines()))
h = r[0]
jx = {k: i for i, k in enumerate(h)}
traffic = {}
with open(os.path.join(out_dir, f"{tag}_ncu_full.txt"), "w") as f:
    f.write(f"# ncu --set full --clock-control none capture: {rep}\n")
    f.write("# phase | us | dram read MB | dram write MB | dram% | sm% | l1% | l2% | warps% | regs | grid\n")
    for row in r[2:]:
        nm = row[jx["Kernel Name"]].split("(")[0].replace("void ", "")
        grid = row[jx["Grid Size"]] if "Grid Size" in jx else ""
        ph = phase_of(nm, grid)
        g = lambda k: float(row[jx[k]].replace(",", ""))
        tu = r[1][jx["gpu__time_duration.sum"]].lower()
        us = g("gpu__time_duration.sum") * {"ns": 1e-3, "nsecond": 1e-3, "ms": 1e3, "msecond": 1e3, "s": 1e6,
                                             "second": 1e6}.get(tu, 1.0)
        rd, wr = g("dram__bytes_read.sum"), g("dram__bytes_write.sum")
        units = r[1]
        u = units[jx["dram__bytes_read.sum"]].lower()
        scale = {"gbyte": 1e9, "mbyte": 1e6, "kbyte": 1e3}.get(u, 1.0)   # -> bytes
        traffic.setdefault(ph, (rd + wr) * scale)
        rd, wr = rd * scale / 1e6, wr * scale / 1e6                        # MB in the table
        f.write(f"{ph:16s} | {us:7.1f} | {rd:8.1f} | {wr:8.1f} | {g(M[3]):5.1f} | {g(M[4]):5.1f} | {g(M[5]):5.1f} | "
                f"{g(M[6]):5.1f} | {g(M[7]):5.1f} | {g(M[8]):4.0f} | {grid}  {nm}\n")
json.dump(traffic, open(os.path.join(out_dir, f"traffic_cfg{cfg}.json"), "w"), indent=1)
print(open(os.path.join(out_dir, f"{tag}_ncu_full.txt")).read())
