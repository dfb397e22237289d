"""Place each kernel of one IB-GM step on the fp64 roofline: executed fp64 flops per
launch (ncu sass op counts: DFMA = 2, DADD/DMUL = 1), DRAM bytes, time; against the
measured fp64 FMA peak (tools/fp64_micro.cu) and HBM peak (MEASURED_PEAKS.json).
  python tools/fp64_ridge.py FP64_MICRO.jsonl NCU.csv CELLS HBM_GBS
"""
import csv
import json
import sys

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.abspath(__file__)))
from kernel_phase import phase_of  # noqa: E402  (the bench line's phase names)

micro, ncsv, cells, hbm = sys.argv[1], sys.argv[2], float(sys.argv[3]), float(sys.argv[4])
peak = max(json.loads(l)["fp64_fma_tflops"] for l in open(micro) if l.startswith("{"))
rows = [r for r in csv.reader(open(ncsv)) if len(r) > 10]
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
SC = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
      "second": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
k = {}
for r in rows[1:]:
    key = (r[ix["ID"]], r[ix["Kernel Name"]].split("(")[0].replace("void ", ""), r[ix["Grid Size"]])
    unit = r[ix["Metric Unit"]].lower()
    v = float(r[ix["Metric Value"]].replace(",", "")) * SC.get(unit, 1.0)
    k.setdefault(key, {})[r[ix["Metric Name"]]] = v
ridge = peak * 1e12 / (hbm * 1e9)
print(f"# fp64 FMA peak {peak:.2f} TFLOP/s (tools/fp64_micro.cu), HBM {hbm:.1f} GB/s -> ridge {ridge:.2f} flop/B")
print("# phase | us | fp64 flop/cell | DRAM B/cell | flop/B | fp64 TFLOP/s | of fp64 peak | fp64 pipe % | HBM frac (ncu bytes)")
for (i, nm, grid), m in sorted(k.items(), key=lambda x: int(x[0][0])):
    t = m["gpu__time_duration.sum"]
    fl = 2 * m["sm__sass_thread_inst_executed_op_dfma_pred_on.sum"] + m["sm__sass_thread_inst_executed_op_dadd_pred_on.sum"] \
        + m["sm__sass_thread_inst_executed_op_dmul_pred_on.sum"]
    by = m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
    ph = phase_of(nm, grid)
    print(f"{ph:14s} | {t * 1e6:8.1f} | {fl / cells:7.1f} | {by / cells:6.1f} | {fl / max(by, 1):6.2f} | "
          f"{fl / t / 1e12:6.2f} | {fl / t / 1e12 / peak:5.2f} | "
          f"{m['sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active']:5.1f} | {by / t / 1e9 / hbm:5.2f}")
