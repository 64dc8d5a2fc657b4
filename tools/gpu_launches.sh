#!/bin/bash
# per-launch breakdown of one config's step: filter-round diagnostics + an ncu launch list
TAG=${TAG:-launches}; CFG=${CFG:-C5}
OUT=gpurun_out/$TAG; mkdir -p $OUT
python build.py > $OUT/build.log 2>&1 || { echo build failed; exit 1; }
MAPSQ_DEBUG=1 timeout 600 python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/plain.json 2> $OUT/plain.err && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
  python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $OUT/ncu.log 2>&1
echo "ncu rc=$?"
grep "filter round" $OUT/plain.err | tail -8
python tools/ncu_launch_seq.py $OUT/launches.csv ${LAST:-60}
