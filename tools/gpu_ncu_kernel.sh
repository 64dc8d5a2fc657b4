#!/bin/bash
# One ncu --set full capture of a kernel family in a bench config, exported as CUDA-line source
# attribution + details (run via gpurun):  CFG=C5 K=expand_kernel SKIP=0 COUNT=1 bash tools/gpu_ncu_kernel.sh
CFG=${CFG:-C5}; K=${K:-expand_kernel}; OUT=gpurun_out/ncuk_${CFG}_$K
mkdir -p $OUT
python build.py > $OUT/build.log 2>&1 || { echo build failed; exit 1; }
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
$CMD > $OUT/plain.log 2>&1 || { echo "plain run failed"; tail -5 $OUT/plain.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" \
  --launch-skip ${SKIP:-0} --launch-count ${COUNT:-1} -o $OUT/rep -f $CMD > $OUT/ncu.log 2>&1
echo "ncu exit $?"
ncu -i $OUT/rep.ncu-rep --page source --csv --print-source cuda > $OUT/source_cuda.csv 2>/dev/null
ncu -i $OUT/rep.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
ncu -i $OUT/rep.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
rm -f $OUT/rep.ncu-rep
gzip -f $OUT/*.csv
