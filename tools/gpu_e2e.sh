python build.py > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out/e2e; rm -f gpurun_out/e2e/*
timeout 900 python -m pytest tests/test_gpu_index.py tests/test_gpu_parity.py -x -q > gpurun_out/e2e/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/e2e/pytest.log
for c in C5 C3 C2 C1; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/e2e/bench_$c.json 2> gpurun_out/e2e/bench_$c.err
  echo "$c rc=$?"; python -c "
import json; d=json.loads(open('gpurun_out/e2e/bench_$c.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e'])"
done
