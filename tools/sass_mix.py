"""Dynamic SASS opcode mix of one kernel from an ncu report (source page).
    python tools/sass_mix.py report.ncu-rep sweep_x [cells]"""
import collections
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
cells = float(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if "Address" in r and "Source" in r)
start = rows.index(hdr) + 1
si, ei = hdr.index("Source"), hdr.index("Thread Instructions Executed")
sti = hdr.index("Warp Stall Sampling (All Samples)")
mix, stalls, seen = collections.Counter(), collections.Counter(), set()
for r in rows[start:]:
    if len(r) <= ei or r[hdr.index("Address")] in seen:
        continue
    seen.add(r[hdr.index("Address")])
    src = r[si].strip()
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    op = op.split(".")[0]
    try:
        mix[op] += int(r[ei] or 0)
        stalls[op] += int(r[sti] or 0)
    except ValueError:
        pass
tot = sum(mix.values())
st = sum(stalls.values())
print(f"total thread-instr {tot:.4g}" + (f" = {tot / cells:.1f} per cell" if cells else ""))
for op, n in mix.most_common(32):
    print(f"{op:10s} {n / (cells or 1):9.1f} {100 * n / tot:5.1f}%  stall {100 * stalls[op] / max(st, 1):5.1f}%")
