"""Opcode mix (warp-level instructions executed) of an ncu report's kernel, from the SASS source page."""
import collections, csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
r = csv.reader(out[1:]); h = next(r); ix = {k: i for i, k in enumerate(h)}
cnt = collections.Counter(); full = collections.Counter()
for row in r:
    s = row[ix["Source"]].strip()
    if not s: continue
    parts = s.split()
    op = parts[1] if parts[0].startswith("@") else parts[0]
    n = int(row[ix["Instructions Executed"]] or 0)
    cnt[op.split(".")[0]] += n; full[op] += n
tot = sum(cnt.values())
print(f"total {tot/1e6:.1f}M warp instructions")
for k, v in cnt.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 30): print(f"  {k:12s} {v/1e6:8.1f}M {100*v/tot:5.1f}%")
