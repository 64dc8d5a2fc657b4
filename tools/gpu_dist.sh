# distributed path at world size 1 on one GPU: the dist GPU tests, and the bench's dist path
# (mapsq_query_dist_indexed / mapsq_join_dist through torchrun, --force-dist) for C5, C3 and C4
python build.py > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out/dist; rm -f gpurun_out/dist/*
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "dist or partition or virtual" > gpurun_out/dist/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/dist/pytest.log
for c in C5 C3 C4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
    bench.py --gpus 1 --force-dist --config $c --steps 5 --warmup 3 > gpurun_out/dist/bench_$c.json 2> gpurun_out/dist/bench_$c.err
  echo "bench $c rc=$?"; tail -3 gpurun_out/dist/bench_$c.err | grep -v NCCL
done
python - <<'PY'
import json
for c in ("C5", "C3", "C4"):
    try:
        d = json.loads(open(f"gpurun_out/dist/bench_{c}.json").read().strip().splitlines()[-1])
    except Exception as e:
        print(c, "no line", e); continue
    print(c, round(d["ms_per_step"], 3), "%.3g" % d["value"], {k: round(v["avg_ms"] * v["launches"] / d["steps"], 3) for k, v in d["kernels"].items()})
PY
