"""Summarise an ncu --set full report: key throughput metrics, stall reasons, hot SASS."""
import csv, subprocess, sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg.per_second",
        "smsp__inst_executed.sum"]
for r in rows[2:]:
    for h in want:
        if h in hdr:
            print(f"  {h:70s} {r[hdr.index(h)]} {units[hdr.index(h)]}")
    for i, h in enumerate(hdr):
        if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
            try:
                if float(r[i]) > 0.05:
                    print(f"  {h:70s} {r[i]}")
            except ValueError:
                pass
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(src.splitlines()))
hi = next(i for i, r in enumerate(srows) if "Source" in r and "Warp Stall Sampling (All Samples)" in r)
h = srows[hi]
isrc, ist = h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = []
for r in srows[hi + 1:]:
    if len(r) > ist:
        try:
            data.append((r[isrc], int(r[ist] or 0)))
        except ValueError:
            pass
tot = sum(n for _, n in data) or 1
c = Counter()
for s, n in data:
    toks = s.split()
    op = toks[1] if toks and toks[0].startswith("@") and len(toks) > 1 else (toks[0] if toks else "?")
    c[op.split(".")[0]] += n
print("  stall samples by opcode:", ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in c.most_common(12)))
print("  hottest SASS:")
for s, n in sorted(data, key=lambda d: -d[1])[:10]:
    print(f"    {100 * n / tot:5.1f}%  {s[:80]}")
