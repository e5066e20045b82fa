"""Instructions executed and warp-stall samples of one kernel in an ncu report, aggregated by CUDA source line
(read here, no GPU). Usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv, subprocess, sys, io, os
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass,cuda"],
                     capture_output=True, text=True).stdout
cur = None; hdr = None; agg = {}
stall_cols = []
for r in csv.reader(io.StringIO(raw)):
    if len(r) == 2 and r[0] == "File Path": cur = r[1]; continue
    if r and r[0] == "Line No":
        hdr = {h: i for i, h in enumerate(r)}
        stall_cols = [h for h in r if h.startswith("stall_") and "Not Issued" not in h]
        continue
    if hdr and cur and len(r) >= len(hdr) - 2:
        try:
            ln = int(r[0]); ie = float(r[hdr["Instructions Executed"]]); st = float(r[hdr["Warp Stall Sampling (All Samples)"]])
        except (ValueError, IndexError):
            continue
        a = agg.setdefault((cur, ln), [0.0, 0.0, {}])
        a[0] += ie; a[1] += st
        for c in stall_cols:
            try: v = float(r[hdr[c]])
            except (ValueError, IndexError): v = 0.0
            if v: a[2][c] = a[2].get(c, 0.0) + v
ti = sum(a[0] for a in agg.values()) or 1; ts = sum(a[1] for a in agg.values()) or 1
print(f"total warp instructions {ti:.3g}, stall samples {ts:.0f}")
tot_st = {}
for a in agg.values():
    for c, v in a[2].items(): tot_st[c] = tot_st.get(c, 0.0) + v
print("stall mix:", ", ".join(f"{c[6:]} {100 * v / ts:.0f}%" for c, v in sorted(tot_st.items(), key=lambda kv: -kv[1])[:8]))
cache = {}
for (f, ln), a in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    if f not in cache:
        cache[f] = open(f).read().splitlines() if os.path.exists(f) else []
    line = cache[f][ln - 1].strip()[:80] if ln - 1 < len(cache[f]) else ""
    why = ",".join(f"{c[6:]}:{100 * v / max(a[1], 1):.0f}" for c, v in sorted(a[2].items(), key=lambda kv: -kv[1])[:3])
    print(f"{100 * a[1] / ts:5.1f}% stall {100 * a[0] / ti:5.1f}% inst  {os.path.basename(f)}:{ln}  [{why}]  {line}")
