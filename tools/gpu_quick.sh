# quick GPU check: semi-join/parity/index tests, C5 per-join diagnostics, C4/C5 with the filter on/off
python build.py > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out/q3; rm -f gpurun_out/q3/*
timeout 900 python -m pytest tests/test_gpu_semijoin.py tests/test_gpu_parity.py tests/test_gpu_index.py -x -q > gpurun_out/q3/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/q3/pytest.log
python tools/diag_query.py C5 10000
for c in C4 C5; do for sj in auto off; do timeout 600 python bench.py --config $c --semijoin $sj --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['workload'], d['config']['semijoin_filter'], d['ms_per_step'], '%.3g'%d['value'], {k:round(v['avg_ms']*v['launches']/5,3) for k,v in d['kernels'].items()})"; done; done
