#!/bin/bash
# ncu --set full capture of the step's main kernels (first occurrence of each), one config.
# Run only after the same bench command exited 0 on this build (the plain run comes first).
TAG=${TAG:-ncufull}; CFG=${CFG:-C5}
OUT=gpurun_out/$TAG; mkdir -p $OUT
KRX=${KRX:-"radix_pass|find_groups|expand_kernel|sj_probe_stage|cfilter_build|filter_build|verify_emit|sj_gather|sj_set_words|pack_hist"}
python build.py > $OUT/build.log 2>&1 || { echo build failed; exit 1; }
CMD="python bench.py --config $CFG --steps 1 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > $OUT/plain.json 2> $OUT/plain.err && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$KRX" \
  --launch-count ${COUNT:-40} -o $OUT/full -f $CMD > $OUT/ncu.log 2>&1
echo "ncu rc=$?"; tail -3 $OUT/ncu.log
ncu -i $OUT/full.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
python tools/ncu_summary.py $OUT/raw.csv > $OUT/summary.md 2>&1; head -60 $OUT/summary.md
for k in ${SRC:-sj_probe_stage find_groups verify_emit}; do
  ncu -i $OUT/full.ncu-rep --page source --csv --kernel-name regex:$k --launch-count 1 > $OUT/source_$k.csv 2>/dev/null
done
gzip -f $OUT/*.csv
rm -f $OUT/full.ncu-rep
