# every bench line of the refresh (no pytest, no ncu): gpurun_out/$1/
OUT=gpurun_out/${1:-benches}; mkdir -p $OUT
python build.py > $OUT/build.log 2>&1 || exit 1
for c in C5 C4 C3 C2 C1; do timeout 600 python bench.py --config $c > $OUT/bench_$c.json 2> $OUT/bench_$c.err; echo "$c exit $?"; done
timeout 600 python bench.py --store scan --no-cpu-baseline > $OUT/bench_C5_scan.json 2> $OUT/bench_C5_scan.err
timeout 600 python bench.py --semijoin off --no-cpu-baseline --no-e2e > $OUT/bench_C5_nofilter.json 2> $OUT/bench_C5_nofilter.err
timeout 600 python bench.py --config C4 --semijoin off --no-cpu-baseline > $OUT/bench_C4_nofilter.json 2> $OUT/bench_C4_nofilter.err
timeout 600 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err; echo "default exit $?"
timeout 600 python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err; echo "ref exit $?"
