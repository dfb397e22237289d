"""Per-source-line totals (instructions executed, warp-stall samples) of one kernel in an
ncu report: ncu -i REP --page source --csv --print-source cuda,sass -k regex:KERNEL.

  python tools/ncu_src_lines.py REP KERNEL_REGEX [top]
"""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Line No")
ie = hdr.index("Instructions Executed")
ws = hdr.index("Warp Stall Sampling (All Samples)")
inst, stall, text = collections.Counter(), collections.Counter(), {}
cur = None
for r in rows[rows.index(hdr) + 1:]:
    if len(r) < len(hdr):
        continue
    if r[0] and not r[0].isdigit():
        continue
    if r[0]:
        cur = int(r[0]); text[cur] = r[1].strip()
    if cur is None:
        continue
    try:
        inst[cur] += float(r[ie] or 0)
        stall[cur] += float(r[ws] or 0)
    except ValueError:
        pass
ti, ts = sum(inst.values()) or 1, sum(stall.values()) or 1
print(f"# {kern}: {ti:.3g} warp instructions, {ts:.0f} stall samples")
for ln in sorted(stall, key=lambda k: -stall[k])[:top]:
    print(f"{100 * inst[ln] / ti:5.1f}% inst {100 * stall[ln] / ts:5.1f}% stall  L{ln}: {text.get(ln, '')[:100]}")
