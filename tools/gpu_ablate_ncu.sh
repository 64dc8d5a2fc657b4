#!/bin/bash
# build-time ablation with DRAM traffic: for each -D set in $VARIANTS (';'-separated), rebuild,
# time $CFG, then one ncu capture of kernel $K (dram bytes, duration).  Output: stdout.
IFS=';' read -ra VS <<< "${VARIANTS}"
for v in "" "${VS[@]}"; do
  MAPSQ_NVCC_DEFS="$v" python build.py --force > /dev/null 2>&1 || { echo "build failed: $v"; continue; }
  timeout 600 python bench.py --config ${CFG:-C5} --no-cpu-baseline --no-e2e > gpurun_out/abl.json 2>/dev/null
  python - "$v" <<'PY'
import json, sys
d = json.loads([l for l in open("gpurun_out/abl.json") if l.startswith("{")][-1])
ks = {k: round(v["avg_ms"] * v["launches"] / d["steps"], 3) for k, v in d["kernels"].items()}
print(f"[{sys.argv[1] or 'default'}] {d['ms_per_step']:.3f} ms", {k: ks[k] for k in sorted(ks, key=lambda k: -ks[k])[:6]})
PY
  timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:"${K:-verify_emit}" --launch-skip ${SKIP:-0} --launch-count 1 --csv python bench.py --config ${CFG:-C5} --steps 1 --warmup 1 --no-cpu-baseline --no-e2e 2>/dev/null | grep -E "dram__bytes|gpu__time" | awk -F'","' '{print "   ", $(NF-2), $(NF-1), $NF}'
done
MAPSQ_NVCC_DEFS="" python build.py --force > /dev/null 2>&1
