# A/B timing of library variants (tools/build_variants.sh): per-call
# timeline of each, plus the default build. usage: ab.sh NAME... [-- timeline args]
set -x
mkdir -p gpurun_out
python tools/gpu/timeline.py $TL_ARGS > gpurun_out/ab_default.json 2>&1
for v in "$@"; do
  CHGPU_LIB=build/variants/libchgpu_$v.so python tools/gpu/timeline.py $TL_ARGS > gpurun_out/ab_$v.json 2>&1
done
python - "$@" <<'PY'
import json, sys
for v in ["default"] + sys.argv[1:]:
    try:
        d = json.load(open(f"gpurun_out/ab_{v}.json"))
    except Exception as e:
        print(v, "FAILED", open(f"gpurun_out/ab_{v}.json").read()[-400:]); continue
    s = d["stages_median"]
    print(f"{v:12s} wall {d['wall_ms_median']:.4f} tot {d['t_total_median']:.4f} " +
          " ".join(f"{k[2:-3]}={v*1e3:.1f}" for k, v in s.items() if v > 0) + f" cand={d['cand']}")
PY
