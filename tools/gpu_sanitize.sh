#!/bin/bash
# compute-sanitizer evidence, ONE tool per gpurun call: TOOL=memcheck|racecheck|synccheck
TOOL=${TOOL:-memcheck}
OUT=gpurun_out/sanitize; mkdir -p $OUT
python build.py > $OUT/build.log 2>&1 || { echo build failed; exit 1; }
timeout 600 python tools/sanitize_run.py > $OUT/plain_$TOOL.log 2>&1 || { echo "plain run failed"; tail $OUT/plain_$TOOL.log; exit 1; }
timeout 2400 compute-sanitizer --tool $TOOL --print-limit 50 python tools/sanitize_run.py > $OUT/$TOOL.log 2>&1
echo "$TOOL rc=$?"; tail -5 $OUT/$TOOL.log
