python build.py > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out/ncu_part; rm -f gpurun_out/ncu_part/*
timeout 900 ncu --set full --clock-control none -k regex:partition_ -s 8 -c 4 -o gpurun_out/ncu_part/part \
  python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --force-dist --config C5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_part/log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/ncu_part/log
ncu -i gpurun_out/ncu_part/part.ncu-rep --page raw --csv > gpurun_out/ncu_part/raw.csv 2>&1
ncu -i gpurun_out/ncu_part/part.ncu-rep --page details --csv > gpurun_out/ncu_part/details.csv 2>&1
rm -f gpurun_out/ncu_part/part.ncu-rep
