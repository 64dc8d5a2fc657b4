#!/bin/bash
# build-time ablation: for each -D set in $VARIANTS (separated by ';'), rebuild libmapsq.so and time
# the given configs (per-kernel ms/step).  e.g. VARIANTS="-DMAPSQ_G_ITEMS=16;-DMAPSQ_G_ITEMS=64"
IFS=';' read -ra VS <<< "${VARIANTS}"
for v in "" "${VS[@]}"; do
  MAPSQ_NVCC_DEFS="$v" python build.py --force > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  for c in ${CONFIGS:-C5}; do
    timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > gpurun_out/abl.json 2>/dev/null
    python - "$v" $c <<'PY'
import json, sys
d = json.loads([l for l in open("gpurun_out/abl.json") if l.startswith("{")][-1])
ks = {k: round(v["avg_ms"] * v["launches"] / d["steps"], 3) for k, v in d["kernels"].items()}
print(f"[{sys.argv[1] or 'default'}] {sys.argv[2]} {d['ms_per_step']:.3f} ms", {k: ks[k] for k in sorted(ks, key=lambda k: -ks[k])[:8]})
PY
  done
done
MAPSQ_NVCC_DEFS="" python build.py --force > /dev/null 2>&1
