"""Per-kernel stall-reason totals and the hottest SASS lines from an ncu report
(source page; needs -lineinfo and --import-source at capture)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
which = int(sys.argv[2]) if len(sys.argv) > 2 else 0
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
blocks, cur = [], []
for line in txt.splitlines():
    if line.startswith('"Kernel Name"'):
        if cur:
            blocks.append(cur)
        cur = [line]
    else:
        cur.append(line)
blocks.append(cur)
b = blocks[which]
rows = list(csv.reader(io.StringIO("\n".join(b[1:]))))
hdr, data = rows[0], rows[1:]
ix = {h: i for i, h in enumerate(hdr)}
cats = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {c: sum(int(r[ix[c]] or 0) for r in data) for c in cats}
allv = sum(tot.values())
print(b[0][:140])
print("total samples", allv)
for c, v in sorted(tot.items(), key=lambda x: -x[1])[:10]:
    print(f"  {c:28s} {v:7d} {100.0 * v / max(allv, 1):5.1f}%")
S = ix["Warp Stall Sampling (All Samples)"]
for r in sorted(data, key=lambda r: -int(r[S] or 0))[:12]:
    top = sorted(((c, int(r[ix[c]] or 0)) for c in cats), key=lambda x: -x[1])[:2]
    print(f"  {r[S]:>6} {r[ix['Source']][:60]:60s} {top}")
