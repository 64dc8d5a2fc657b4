#!/bin/bash
# A/B of the filter's carried columns (MAPSQ_SJ_CARRY 0 / 1 / 2=auto) on C5, C4, C3, C2: per-kernel
# times per setting, plus one MAPSQ_DEBUG run of C5 (filter rounds).  Output in gpurun_out/$TAG.
TAG=${TAG:-carry}
OUT=gpurun_out/$TAG
mkdir -p $OUT; rm -f $OUT/*
python build.py > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
if [ "${TESTS:-1}" = 1 ]; then
  timeout 900 python -m pytest tests/test_gpu_semijoin.py tests/test_gpu_parity.py -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
  timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q > $OUT/pytest_full.log 2>&1; echo "full pytest rc=$?"; tail -2 $OUT/pytest_full.log
fi
MAPSQ_DEBUG=1 python bench.py --config C5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2> $OUT/debug_C5.err
grep mapsq $OUT/debug_C5.err | head -12
for c in ${CONFIGS:-C5 C4 C3 C2}; do
  for m in 0 1 2; do
    MAPSQ_SJ_CARRY=$m timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $OUT/bench_${c}_$m.json 2> $OUT/bench_${c}_$m.err
    python - $OUT/bench_${c}_$m.json $m <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read())
print(d["config"]["workload"], "carry", sys.argv[2], round(d["ms_per_step"], 3), "%.3g" % d["value"])
for k, v in d["kernels"].items():
    print("   %-16s %3d %.3f ms/step" % (k, v["launches"], v["avg_ms"] * v["launches"] / d["steps"]))
PY
  done
done
