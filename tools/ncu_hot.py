"""Hottest source lines of one kernel in an ncu report (read here, no GPU):
warp-stall samples per SASS line with the CUDA source line they map to.
Usage: python tools/ncu_hot.py report.ncu-rep kernel_regex [top]"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}",
                      "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = None
out = []
for r in rows:
    if "Warp Stall Sampling (All Samples)" in r:
        hdr = {h: i for i, h in enumerate(r)}
        continue
    if hdr and len(r) == len(hdr):
        try:
            s = float(r[hdr["Warp Stall Sampling (All Samples)"]])
        except ValueError:
            continue
        out.append((s, r[hdr["Source"]][:110]))
tot = sum(s for s, _ in out) or 1
for s, src in sorted(out, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}%  {src}")
