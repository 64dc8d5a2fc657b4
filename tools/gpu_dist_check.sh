#!/bin/bash
# multi-rank checks on one GPU: 2/3-process library exchange tests, world-1 NCCL dist bench
OUT=gpurun_out/${TAG:-d1}; mkdir -p $OUT
python build.py > $OUT/build.log 2>&1 || { tail $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_dist2.py -x -q > $OUT/pytest_dist2.log 2>&1; echo "dist2 rc=$?"; tail -30 $OUT/pytest_dist2.log
if [ "${FAST:-1}" = 1 ]; then
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > $OUT/pytest_fast.log 2>&1; echo "fast rc=$?"; tail -3 $OUT/pytest_fast.log
fi
for c in ${CONFIGS:-C5}; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --force-dist --config $c --no-cpu-baseline --no-e2e > $OUT/bench_force_dist_$c.json 2> $OUT/bench_force_dist_$c.err; echo "force-dist $c rc=$?"
python - $OUT/bench_force_dist_$c.json <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
print(d["config"]["workload"], round(d["ms_per_step"], 3), "%.3g" % d["value"], "exchange B/step %.3g" % d["exchange"]["bytes_per_step"])
for k, v in d["kernels"].items():
    print("   %-18s %3d %.3f ms/step" % (k, v["launches"], v["avg_ms"] * v["launches"] / d["steps"]))
PY
done
# the bench's N > 1 code path with 2 rank processes on this one GPU (gloo + host collectives;
# a smoke test of the JSON line, not a measurement)
if [ "${BENCH2:-1}" = 1 ]; then
for c in "C3 --univ 50" "C5 --univ 100" "C4 --rows 10000000"; do
  MAPSQ_BENCH_HOSTCOLL=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29544 \
    bench.py --gpus 2 --steps 2 --warmup 1 --no-cpu-baseline --config $c > $OUT/bench2_$(echo $c | cut -d' ' -f1).json 2> $OUT/bench2_$(echo $c | cut -d' ' -f1).err
  echo "bench world-2 (one GPU) $c rc=$?"; tail -c 600 $OUT/bench2_$(echo $c | cut -d' ' -f1).json; tail -2 $OUT/bench2_$(echo $c | cut -d' ' -f1).err
done
fi
