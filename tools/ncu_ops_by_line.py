"""Per-source-line opcode counts (warp instructions executed) of an ncu report:
    python tools/ncu_ops_by_line.py REP [OPS...]"""
import collections
import csv
import subprocess
import sys

src = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
ops_wanted = sys.argv[2:] or ["LDL", "STL", "BSSY", "BRA", "IMAD", "ISETP", "VIMNMX", "LDC"]
cur, curfile = None, None
agg = collections.defaultdict(collections.Counter)
for r in csv.reader(src.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        curfile = r[1].split("/")[-1]
        continue
    if r[0] in ("Line No", "Function Name"):
        continue
    if r[0]:
        cur = (curfile, r[0], r[1].strip()[:80])
        continue
    if len(r) > 7 and r[3].strip() and r[7].isdigit():
        s = r[3].strip()
        op = (s.split()[1] if s.startswith("@") else s.split()[0]).split(".")[0]
        agg[cur][op] += int(r[7])
for op in ops_wanted:
    rows = sorted(((c[op], k) for k, c in agg.items() if c[op] > 0), reverse=True)[:7]
    print(op)
    for n, k in rows:
        print("   %6.1fM %-16s %5s %s" % (n / 1e6, k[0][:16], k[1], k[2][:70]))
