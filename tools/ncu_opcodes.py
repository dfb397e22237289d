"""Executed warp instructions of one kernel in an ncu report, grouped by SASS opcode.

  python tools/ncu_opcodes.py REP KERNEL_REGEX [top]
"""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                      "regex:" + kern], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if r and r[0] == "Address")
ie, src = hdr.index("Instructions Executed"), hdr.index("Source")
cnt = collections.Counter()
for r in rows[rows.index(hdr) + 1:]:
    if len(r) < len(hdr) or not r[0].startswith("0x"):
        continue
    t = r[src].strip().split()
    if not t:
        continue
    op = t[1] if t[0].startswith("@") and len(t) > 1 else t[0]
    try:
        cnt[op.split(".")[0]] += float(r[ie] or 0)
    except ValueError:
        pass
tot = sum(cnt.values()) or 1
print(f"# {kern}: {tot:.4g} warp instructions")
for op, v in cnt.most_common(top):
    print(f"{op:12s} {v:12.4g} {100 * v / tot:5.1f}%")
