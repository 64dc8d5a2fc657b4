mkdir -p gpurun_out/d1
python build.py > gpurun_out/d1/build.log 2>&1 || { tail gpurun_out/d1/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_dist2.py -x -q > gpurun_out/d1/pytest_dist2.log 2>&1; echo "dist2 rc=$?"; tail -30 gpurun_out/d1/pytest_dist2.log
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/d1/pytest_fast.log 2>&1; echo "fast rc=$?"; tail -3 gpurun_out/d1/pytest_fast.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --force-dist --config C5 --no-cpu-baseline > gpurun_out/d1/bench_force_dist.json 2> gpurun_out/d1/bench_force_dist.err; echo "force-dist rc=$?"; cut -c1-600 gpurun_out/d1/bench_force_dist.json
timeout 300 python bench.py --gpus 2 --steps 1 --warmup 1 > gpurun_out/d1/bench_g2.json 2> gpurun_out/d1/bench_g2.err; echo "gpus2 rc=$?"; tail -2 gpurun_out/d1/bench_g2.err
