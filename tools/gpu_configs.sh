# all GPU tests, then every config (and the filter-off variants) with per-kernel times
python build.py > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for c in "C5" "C4" "C3" "C4 --semijoin off" "C5 --semijoin off" "C2" "C1"; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['config']['semijoin_filter'], round(d['ms_per_step'],3), '%.3g'%d['value'], d['roofline']['kernel'], round(d['roofline']['frac'],3), round(d['hbm']['frac_of_peak'],3), {k:round(v['avg_ms']*v['launches']/5,3) for k,v in d['kernels'].items()})"; done
