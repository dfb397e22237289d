"""Summarise `nvcc -Xptxas -v` output: kernel, registers, stack, spill bytes."""
import re, subprocess, sys
src = sys.argv[1]
flt = sys.argv[2] if len(sys.argv) > 2 else ""
out = subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
                      "-Xcompiler", "-fPIC", "-c", "-o", "/dev/null", src, "-Xptxas", "-v"],
                     capture_output=True, text=True).stderr
cur = None
rows = []
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = subprocess.run(["cu++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        cur = re.sub(r"\(ibgm::LineCoef.*|\(const double.*|\(ibgm::Ctx.*|\(int.*", "", cur.replace("ibgm::", "").replace("void ", "").replace("(int)", ""))
        st = sp = 0
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores", line)
    if m and cur:
        st, sp = int(m.group(1)), int(m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        rows.append((cur, int(m.group(1)), st, sp))
        cur = None
for r in rows:
    if flt in r[0]:
        print(f"{r[0]:55s} regs={r[1]:4d} stack={r[2]:5d} spill={r[3]:5d}")
