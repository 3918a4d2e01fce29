# Per-kernel durations (ncu, serialised) of a few steps of the 20M uniform
# timeline; prints name + microseconds for the last N launches.
N=${N:-12}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c ${C:-80} --csv \
  --log-file gpurun_out/launches_tl.csv python tools/gpu/timeline.py ${ARGS:-} > /dev/null 2>&1
python - <<'PY'
import csv, os
rows = list(csv.reader(open("gpurun_out/launches_tl.csv")))
h = next(r for r in rows if r and r[0] == "ID")
ix = {c: i for i, c in enumerate(h)}
out = [(r[ix["Kernel Name"]].split("(")[0].split("::")[-1], float(r[ix["Metric Value"]]) / 1e3)
       for r in rows if r and r[0].isdigit() and len(r) == len(h)]
n = int(os.environ.get("N", "12"))
for name, us in out[-n:]:
    print(f"{name:28s} {us:8.2f} us")
PY
