"""Instructions executed and stall samples per CUDA source line of one
kernel: ncu's SASS page (in address order) zipped with nvdisasm's line
table of the same cubin. usage: ncu_lines.py REPORT CUBIN FUNC [N]"""
import collections, csv, io, re, subprocess, sys
rep, cubin, func = sys.argv[1:4]
n = int(sys.argv[4]) if len(sys.argv) > 4 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
i = next(k for k, r in enumerate(rows) if r and r[0] == "Address")
h = rows[i]
ix = {c: h.index(c) for c in h}
sass = [(int(r[ix["Instructions Executed"]] or 0), int(r[ix["Warp Stall Sampling (All Samples)"]] or 0), r[ix["Source"]].strip())
        for r in rows[i + 1:]]
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
line = None
lines = []
inside = False
for l in dis.splitlines():
    if l.startswith(".text.") or re.match(r"\s*\.section\s+\.text\.", l):
        inside = func in l
        continue
    if not inside:
        continue
    m = re.search(r'//## File ".*?/([^/"]+)", line (\d+)', l)
    if m:
        line = f"{m.group(1)}:{m.group(2)}"
        continue
    if re.match(r"\s*/\*[0-9a-f]{4,}\*/", l):
        lines.append(line)
print(f"sass rows {len(sass)}, disasm instructions {len(lines)}")
agg = collections.defaultdict(lambda: [0, 0])
for (exe, st, _), ln in zip(sass, lines):
    agg[ln][0] += exe
    agg[ln][1] += st
tot = sum(v[0] for v in agg.values()) or 1
tst = sum(v[1] for v in agg.values()) or 1
for ln, (exe, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{ln:24s} inst {exe / tot * 100:5.1f}%  stall {st / tst * 100:5.1f}%")
