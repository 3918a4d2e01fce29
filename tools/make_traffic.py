"""profiles/<round>/traffic.json from ncu --set full captures: per-launch
DRAM bytes (dram__bytes_read.sum + dram__bytes_write.sum) of each kernel,
keyed like bench.py's per_kernel (combined stages sum their kernels).

usage: python tools/make_traffic.py OUT.json REPORT.ncu-rep ..."""
import csv
import io
import json
import subprocess
import sys

KERNELS = {"k_extremes_partial": "k1_extremes", "k_classify_survivors": "k2_classify_survivors",
           "k_classify_compact": "k2_classify_compact", "k_bin_scan": "k3_bin_scan",
           "k_filter": "k3_filter", "k_spa_small": "k4_spa_small", "k_spa_finish": "k4_spa_finish"}
STAGES = {"k1k2_discard": ["k1_extremes", "k2_classify_survivors"],
          "k4_chunk_spa": ["k4_spa_small", "k4_spa_finish"]}

out = {}
for rep in sys.argv[2:]:
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units, r = rows[0], rows[1], rows[2]
    name = r[h.index("Kernel Name")]
    base = name.split("(")[0].split("::")[-1].split("<")[0].split()[-1]

    def val(m):
        v = float(r[h.index(m)].replace(",", ""))
        return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[h.index(m)], 1)

    if base in KERNELS:
        out[KERNELS[base]] = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
for stage, parts in STAGES.items():
    if all(p in out for p in parts):
        out[stage] = sum(out[p] for p in parts)
json.dump(out, open(sys.argv[1], "w"), indent=1)
print(out)
