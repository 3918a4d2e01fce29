"""profiles/round1/traffic.json from ncu --set full captures: per-launch
DRAM bytes (read + write) of each kernel, keyed like bench.py's per_kernel."""
import csv, io, json, subprocess, sys

KEYS = {"k_classify_survivors": "k2_classify_survivors", "k_filter": "k3_filter",
        "k_extremes_partial": "k1_extremes", "k_bin_scan": "k3_bin_scan",
        "k_spa_chunks": "k4_spa_chunks", "k_spa_emit": "k4_spa_emit",
        "k_bin_sort_warp": "k3_bin_sort", "k_classify_compact": "k2_classify_compact"}
out = {}
for rep in sys.argv[2:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, r = rows[0], rows[1], rows[2]
    name = r[h.index("Kernel Name")]
    def val(m):
        v = float(r[h.index(m)].replace(",", ""))
        u = units[h.index(m)]
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    b = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
    for k, key in KEYS.items():
        if name.startswith(k) or name.split("(")[0].split()[-1].startswith(k) or f" {k}(" in f" {name}":
            out[key] = b
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(out)
