#!/bin/bash
# Round evidence refresh on a B200 box (run via gpurun from the repo root):
#   gpu tests, bench lines for every config + the reference arm, the C5 ncu launch list and one
#   ncu --set full capture of the step's kernels. Output under gpurun_out/$TAG/.
TAG=${1:-refresh}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python build.py > $OUT/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
for c in C5 C4 C3 C2 C1; do
  timeout 600 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  echo "$c exit $?"; cat $OUT/bench_$c.json | cut -c1-200
done
# the same with the full-table scan and with the semi-join filter off (for the record)
timeout 600 python bench.py --store scan --no-cpu-baseline > $OUT/bench_C5_scan.json 2> $OUT/bench_C5_scan.err
timeout 600 python bench.py --semijoin off --no-cpu-baseline --no-e2e > $OUT/bench_C5_nofilter.json 2> $OUT/bench_C5_nofilter.err
timeout 600 python bench.py --config C4 --semijoin off --no-cpu-baseline > $OUT/bench_C4_nofilter.json 2> $OUT/bench_C4_nofilter.err
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
echo "ref exit $?"
if [ "${NCU:-1}" = 1 ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file $OUT/ncu_launches_C5.csv python bench.py --steps 1 --warmup 3 --no-e2e \
    --no-cpu-baseline > $OUT/ncu_l.log 2>&1
  echo "ncu launches exit $?"
  # one full capture of every kernel of one step: skip/count from the launch list (the step ends
  # with residual_expand; the first timed step follows the 3 warm-up steps)
  read SKIP COUNT <<< "$(python - $OUT/ncu_launches_C5.csv <<'PY'
import csv, re, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
ki = rows[hi].index("Kernel Name")
names = [r[ki] for r in rows[hi + 1:] if len(r) > ki]
rx = re.compile("radix_pass|wfilter|filter_|find_groups|expand|residual|pack_hist")
ends = [i for i, n in enumerate(names) if "residual_expand" in n]
start, end = ends[2] + 1, ends[3] + 1
print(sum(bool(rx.search(n)) for n in names[:start]), sum(bool(rx.search(n)) for n in names[start:end]))
PY
)"
  echo "full capture: skip $SKIP count $COUNT"
  timeout 1500 ncu --set full --clock-control none --import-source on \
    -k regex:"radix_pass|wfilter|filter_|find_groups|expand|residual|pack_hist" \
    --launch-skip ${SKIP:-101} --launch-count ${COUNT:-33} -o $OUT/ncu_full_C5 -f \
    python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $OUT/ncu_f.log 2>&1
  echo "ncu full exit $?"
  ncu -i $OUT/ncu_full_C5.ncu-rep --page raw --csv > $OUT/ncu_full_C5_raw.csv 2>/dev/null
  ncu -i $OUT/ncu_full_C5.ncu-rep --page details --csv > $OUT/ncu_full_C5_details.csv 2>/dev/null
  for k in radix_pass cfilter_probe wfilter_probe find_groups; do
    ncu -i $OUT/ncu_full_C5.ncu-rep --page source --csv --kernel-name regex:$k --launch-count 1 \
      > $OUT/ncu_source_$k.csv 2>/dev/null
  done
  gzip -f $OUT/*.csv
  # the report itself is too large to bring back (gpurun_out is capped at 64 MiB)
  rm -f $OUT/ncu_full_C5.ncu-rep
fi
if [ "${ABLATE:-0}" = 1 ] && [ -x tools/radix_ablate ]; then
  timeout 600 tools/radix_ablate zipf 400000000 > $OUT/ablate_zipf.log 2>&1
  timeout 600 tools/radix_ablate 300000000 0.1 1 > $OUT/ablate_rand.log 2>&1
  cat $OUT/ablate_zipf.log $OUT/ablate_rand.log
fi
du -sh $OUT
