python build.py > /dev/null 2>&1
for b in ${BITS:-29 28 27}; do
MAPSQ_SJ_COLBITS=$b MAPSQ_DEBUG=1 timeout 600 python bench.py --config C5 --no-cpu-baseline --no-e2e > gpurun_out/abl_$b.json 2> gpurun_out/abl_$b.err
python - gpurun_out/abl_$b.json $b <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read())
print("bits", sys.argv[2], round(d["ms_per_step"], 3), {k: round(v["avg_ms"] * v["launches"] / d["steps"], 3) for k, v in d["kernels"].items() if k.startswith("filter") or k == "verify_emit"})
PY
grep "filter round" gpurun_out/abl_$b.err | tail -3
done
