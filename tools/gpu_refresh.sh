#!/bin/bash
# Round evidence refresh on a B200 box (run via gpurun from the repo root):
#   every GPU test, bench lines for every config + the reference arm, the C5 / C4 ncu launch
#   lists and one ncu --set full capture of each step's kernels (DRAM traffic per library timer
#   -> profiles/ncu_traffic_<cfg>.json, read by bench.py's roofline "traffic").  Output under
#   gpurun_out/$TAG/.
TAG=${1:-refresh}
OUT=gpurun_out/$TAG
mkdir -p $OUT
python build.py > $OUT/build.log 2>&1 || { echo build failed; exit 1; }
if [ "${TESTS:-1}" = 1 ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
  tail -3 $OUT/pytest_gpu.log
fi
for c in C5 C4 C3 C2 C1; do
  # (the launch-bound small configs: more steps, so a jittery step does not dominate the mean)
  ST=""; [ $c = C1 -o $c = C2 ] && ST="--steps 200 --warmup 20"
  timeout 600 python bench.py --config $c $ST > $OUT/bench_$c.json 2> $OUT/bench_$c.err
  echo "$c exit $?"; cut -c1-160 $OUT/bench_$c.json
done
# the same with the full-table scan and with the semi-join filter off (for the record)
timeout 600 python bench.py --store scan --no-cpu-baseline > $OUT/bench_C5_scan.json 2> $OUT/bench_C5_scan.err
timeout 600 python bench.py --semijoin off --no-cpu-baseline --no-e2e > $OUT/bench_C5_nofilter.json 2> $OUT/bench_C5_nofilter.err
timeout 600 python bench.py --config C4 --semijoin off --no-cpu-baseline > $OUT/bench_C4_nofilter.json 2> $OUT/bench_C4_nofilter.err
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
echo "ref exit $?"
if [ "${NCU:-1}" = 1 ]; then
  for c in C5 C4; do
    CMD="python bench.py --config $c --steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
    $CMD > $OUT/plain_$c.log 2>&1 && \
    timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/ncu_launches_$c.csv $CMD > $OUT/ncu_l_$c.log 2>&1
    echo "ncu launches $c exit $?"
    # full capture of the first step's kernels (the warm-up step: same work)
    timeout 1500 ncu --set full --clock-control none --import-source on \
      -k regex:"radix_pass|filter|sj_|find_groups|expand|verify_emit|pack_hist|small_join" \
      --launch-count ${COUNT:-40} -o $OUT/ncu_full_$c -f $CMD > $OUT/ncu_f_$c.log 2>&1
    echo "ncu full $c exit $?"
    ncu -i $OUT/ncu_full_$c.ncu-rep --page raw --csv > $OUT/ncu_full_${c}_raw.csv 2>/dev/null
    python tools/ncu_summary.py $OUT/ncu_full_${c}_raw.csv $OUT/ncu_traffic_$c.json $([ $c = C4 ] && echo 0 || echo 2) > $OUT/ncu_full_$c.md 2>&1
    for k in sj_probe_stage radix_pass expand_kernel verify_emit find_groups; do
      ncu -i $OUT/ncu_full_$c.ncu-rep --page source --csv --kernel-name regex:$k --launch-count 1 \
        > $OUT/ncu_source_${c}_$k.csv 2>/dev/null
    done
    rm -f $OUT/ncu_full_$c.ncu-rep
  done
  gzip -f $OUT/*.csv
fi
