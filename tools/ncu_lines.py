"""Summarise an ncu report: key metrics, stall reasons, opcode mix and hottest source lines."""
import collections, csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
d = {h: (v, u) for h, u, v in zip(rows[0], rows[1], rows[2])}
keys = ["gpu__time_duration.sum", "smsp__inst_executed.sum", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__thread_inst_executed_per_inst_executed.ratio",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]
for k in keys:
    print(f"{k:70s} {d.get(k)}")
st = []
for h, (v, u) in d.items():
    if "average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio"):
        try:
            st.append((float(v), h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")))
        except ValueError:
            pass
print("stalls/issue:", ", ".join(f"{n} {v:.2f}" for v, n in sorted(st, reverse=True) if v > 0.05))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
per, text, hdr, cur = collections.Counter(), {}, None, None
ops = collections.Counter()
for r in csv.reader(src.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        iE = r.index("Instructions Executed")
        continue
    if hdr is None or r[0] == "Function Name":
        continue
    try:
        ln, n = int(r[0]), int(r[iE] or 0)
    except ValueError:
        continue
    per[(cur, ln)] += n
    text[(cur, ln)] = r[1][:100]
tot = sum(per.values()) or 1
for k, v in per.most_common(top):
    print(f"{100 * v / tot:5.1f}% {k[0]}:{k[1]}  {text[k].strip()}")
