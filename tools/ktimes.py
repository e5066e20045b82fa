"""Per-kernel durations from an ncu --csv launch list (gpu__time_duration.sum):
python tools/ktimes.py launches.csv [last_n]"""
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
rows = rows[next(i for i, r in enumerate(rows) if r[0] == "ID"):]  # skip the program's own output
hdr = rows[0]
ik, iv = hdr.index("Kernel Name"), hdr.index("Metric Value")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
rows = [r for r in rows[1:] if "mumode_gpu" in r[ik]]
for r in rows[-n:]:
    print(f"{float(r[iv].replace(',', '')) / 1000:9.1f} us  {r[ik][:110]}")
