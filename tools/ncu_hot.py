"""Hottest SASS instructions of an ncu report (stall samples, L2 sectors):
python tools/ncu_hot.py REPORT [N]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
i = next(k for k, r in enumerate(rows) if r and r[0] == "Address")
h = rows[i]
ix = {c: h.index(c) for c in h}
data = rows[i + 1:]
tot = sum(int(r[ix["Warp Stall Sampling (All Samples)"]] or 0) for r in data)
data.sort(key=lambda r: -int(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
print(f"total samples {tot}")
for r in data[:n]:
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    print(f"{s / tot * 100:5.1f}% {r[ix['Source']][:60]:60s} L2sect={r[ix['L2 Theoretical Sectors Global']]:>9s} exe={r[ix['Instructions Executed']]}")
