"""Per-CUDA-source-line instruction and stall shares of one kernel in an ncu
report (needs -lineinfo builds and --import-source).
usage: python tools/ncu_lines.py report.ncu-rep kernel-regex [top]"""
import csv
import io
import subprocess
import sys

rep, rx = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass",
                      "--kernel-name", "regex:" + rx], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
fname, hdr, lines = None, None, []
for r in rows:
    if r and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and r and r[0].isdigit():
        try:
            ie = float(r[hdr.index("Instructions Executed")] or 0)
            st = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except ValueError:
            continue
        lines.append((fname, int(r[0]), ie, st, r[1].strip()[:70]))
ti = sum(l[2] for l in lines) or 1
ts = sum(l[3] for l in lines) or 1
print(f"{'file':16s} {'line':>5s} {'instr%':>7s} {'stall%':>7s}")
for l in sorted(lines, key=lambda l: -(l[2] / ti + l[3] / ts))[:top]:
    print(f"{l[0]:16s} {l[1]:5d} {l[2] / ti * 100:6.1f}% {l[3] / ts * 100:6.1f}%  {l[4]}")
