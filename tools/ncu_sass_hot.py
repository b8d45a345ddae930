"""Hot SASS of an ncu report (--page source --print-source sass): every
instruction executed at least MIN times, with executions (millions) and
warp-stall samples, plus the per-opcode totals of the hot region.

    python tools/ncu_sass_hot.py report.ncu-rep [MIN]
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
lo = float(sys.argv[2]) if len(sys.argv) > 2 else 1e6
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ia, isrc, iex, ist = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), \
    h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[2:]:
    try:
        data.append((r[ia], r[isrc].strip(), int(r[iex]), int(r[ist])))
    except (ValueError, IndexError):
        continue
tot = sum(d[2] for d in data)
tst = sum(d[3] for d in data)
print(f"# {rep}: {tot / 1e6:.1f} M warp instructions, {tst} stall samples")
ops = collections.Counter()
for a, s, e, st in data:
    if e >= lo:
        print(f"{a[-6:]} {e / 1e6:6.2f} {st:6d}  {s[:96]}")
    op = s.split()[0] if not s.startswith("@") else s.split()[1]
    ops[op.split(".")[0]] += e
print("# opcode mix (whole kernel, M):", ", ".join(f"{k} {v / 1e6:.0f}" for k, v in ops.most_common(24)))
