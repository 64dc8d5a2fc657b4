python build.py > /dev/null 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_index.py -x -q > gpurun_out/e2e_pytest.log 2>&1; echo "index tests rc=$?"; tail -3 gpurun_out/e2e_pytest.log
for c in C5 C3 C2; do
timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/e2e_$c.json 2> gpurun_out/e2e_$c.err
python - gpurun_out/e2e_$c.json <<'PY'
import json, sys
d = json.loads([l for l in open(sys.argv[1]) if l.startswith("{")][-1])
e = d.get("e2e") or {}
print(d["config"]["workload"], round(d["ms_per_step"], 3), "%.3g" % d["value"], "e2e %.3g" % (e.get("value") or 0), e.get("ms_per_step"), e.get("h2d_bytes_per_step"), e.get("d2h_bytes_per_step"))
PY
done
