"""Summarise an ncu report: per kernel launch time, DRAM bytes, throughputs, occupancy."""
import csv, subprocess, sys
rep = sys.argv[1]
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
     "l1tex__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
     "smsp__average_warp_latency_issue_stalled_long_scoreboard", "smsp__pcsamp_warps_issue_stalled_long_scoreboard",
     "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M)], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
hdr = r[0]
units = r[1]
idx = {h: i for i, h in enumerate(hdr)}
# ncu picks the unit per report (us / ms, Mbyte / Gbyte): normalise to us and MB
SCALE = {"ns": 1e-3, "us": 1.0, "ms": 1e3, "s": 1e6, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "second": 1e6,
         "byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3, "Tbyte": 1e6}
short = {"gpu__time_duration.sum": "us", "dram__bytes_read.sum": "rdMB", "dram__bytes_write.sum": "wrMB",
         "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram%", "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm%",
         "l1tex__throughput.avg.pct_of_peak_sustained_elapsed": "l1%", "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2%",
         "sm__warps_active.avg.pct_of_peak_sustained_active": "warps%", "launch__registers_per_thread": "regs",
         "launch__grid_size": "grid", "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active": "fp64%"}
for row in r[2:]:
    name = row[idx["Kernel Name"]]
    name = name.split("(")[0].replace("void ", "")
    vals = []
    for k, s in short.items():
        if k in idx:
            v = row[idx[k]]
            try:
                v = f"{float(v.replace(',', '')) * SCALE.get(units[idx[k]], 1.0):.1f}"
            except ValueError:
                pass
            vals.append(f"{s}={v}")
    print(f"{name:38s} " + " ".join(vals))
