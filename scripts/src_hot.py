"""Hottest CUDA source lines (warp stall samples) of one kernel in an ncu report."""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 12
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
f, lines, ist = "?", [], None
for r in csv.reader(out.splitlines()):
    if r and r[0] == "File Path":
        f = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        ist = r.index("Warp Stall Sampling (All Samples)")
    elif ist is not None and len(r) > ist and r[0].strip():
        n = int(r[ist]) if r[ist].strip().isdigit() else 0
        lines.append((n, f"{f}:{r[0]}", r[1].strip()[:90]))
tot = sum(n for n, _, _ in lines) or 1
print(kern, "samples", tot)
for n, loc, src in sorted(lines, reverse=True)[:top]:
    print(f"  {100 * n / tot:5.1f}%  {loc:22s} {src}")
