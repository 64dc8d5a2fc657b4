#!/bin/bash
# A/B of an environment knob ($VAR over $VALS, e.g. VAR=MAPSQ_PV VALS="0 1") on the given configs:
# GPU tests first (TESTS=1), then per-kernel times per setting.  Output in gpurun_out/$TAG.
TAG=${TAG:-ab}
OUT=gpurun_out/$TAG
mkdir -p $OUT; rm -f $OUT/*
python build.py > $OUT/build.log 2>&1 || { echo build failed; tail $OUT/build.log; exit 1; }
if [ "${TESTS:-1}" = 1 ]; then
  timeout 900 python -m pytest ${TESTFILES:-tests/test_gpu_parity.py tests/test_gpu_semijoin.py} -x -q > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
  timeout 1200 python -m pytest tests/test_gpu_fullsize.py -x -q > $OUT/pytest_full.log 2>&1; echo "full pytest rc=$?"; tail -2 $OUT/pytest_full.log
fi
for c in ${CONFIGS:-C5 C4 C3 C2}; do
  for m in $VALS; do
    env $VAR=$m timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $OUT/bench_${c}_$m.json 2> $OUT/bench_${c}_$m.err
    python - $OUT/bench_${c}_$m.json "$VAR=$m" <<'PY'
import json, sys
d = json.loads(open(sys.argv[1]).read())
ks = {k: round(v["avg_ms"] * v["launches"] / d["steps"], 3) for k, v in d["kernels"].items()}
print(d["config"]["workload"], sys.argv[2], round(d["ms_per_step"], 3), "%.3g" % d["value"], {k: ks[k] for k in sorted(ks, key=lambda k: -ks[k])[:9]})
PY
  done
done
