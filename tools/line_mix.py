"""Per-source-line SASS opcode counts of one kernel from an ncu report
(-lineinfo builds): python tools/line_mix.py report kernel cells [opcode-prefix ...]"""
import collections
import csv
import re
import subprocess
import sys

rep, kern, cells = sys.argv[1], sys.argv[2], float(sys.argv[3])
ops = sys.argv[4:]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
fname, line, text = "?", "?", ""
per = collections.defaultdict(collections.Counter)
stall = collections.defaultdict(collections.Counter)
src = {}
hdr = None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 9:
        continue
    if r[0]:
        line, text = r[0], r[1]
        src[(fname, line)] = text.strip()[:70]
        continue
    ins = r[3].strip()
    op = ins.split()[1] if ins.startswith("@") else (ins.split()[0] if ins else "?")
    op = op.split(".")[0]
    try:
        n = int(r[8] or 0)
    except ValueError:
        continue
    per[(fname, line)][op] += n
    try:
        stall[(fname, line)][op] += int(r[4] or 0)
    except ValueError:
        pass
by_stall = "--stall" in ops
ops = [o for o in ops if o != "--stall"]
src_tab = stall if by_stall else per
tot = collections.Counter()
for k, c in src_tab.items():
    tot[k] = sum(v for o, v in c.items() if not ops or any(o.startswith(p) for p in ops))
if by_stall:
    cells = sum(tot.values()) / 100.0  # percent of all samples
for k, v in tot.most_common(40):
    if v == 0:
        break
    mix = " ".join(f"{o}:{n / cells:.1f}" for o, n in per[k].most_common(6))
    print(f"{v / cells:7.2f} {k[0]}:{k[1]:>4} {src.get(k, '')[:60]:60s} | {mix}")
