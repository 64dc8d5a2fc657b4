#!/bin/bash
# one build -> test -> bench iteration on a B200 box (via gpurun): fast GPU parity tests, the
# full-size fingerprints, then per-kernel times of the given configs.  Output in gpurun_out/$TAG.
TAG=${TAG:-iter}
OUT=gpurun_out/$TAG
mkdir -p $OUT; rm -f $OUT/*
python build.py > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > $OUT/pytest_fast.log 2>&1; echo "fast pytest rc=$?"; tail -3 $OUT/pytest_fast.log
if [ "${FULL:-1}" = 1 ]; then
  timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q > $OUT/pytest_full.log 2>&1; echo "full pytest rc=$?"; tail -3 $OUT/pytest_full.log
fi
for c in ${CONFIGS:-"C5" "C4"}; do
  timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  python - $OUT/bench_$c.json <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read())
r = d["roofline"]
print(d["config"]["workload"], d["config"].get("semijoin_filter"), round(d["ms_per_step"], 3), "%.3g" % d["value"],
      r["kernel"], round(r["frac"], 3), round(d["hbm"]["frac_of_peak"], 3))
for k, v in d["kernels"].items():
    print("   %-16s %3d %.3f ms/step" % (k, v["launches"], v["avg_ms"] * v["launches"] / d["steps"]))
PY
done
