python build.py > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out/q7; rm -f gpurun_out/q7/*
timeout 900 ncu --set full --import-source on -k regex:"expand_kernel" --launch-skip 9 --launch-count 3 -o gpurun_out/q7/exp -f python bench.py --config C3 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/q7/f.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/q7/exp.ncu-rep --page raw --csv > gpurun_out/q7/raw.csv 2>/dev/null
ncu -i gpurun_out/q7/exp.ncu-rep --page source --csv --launch-skip 2 --launch-count 1 > gpurun_out/q7/src.csv 2>/dev/null
gzip -f gpurun_out/q7/*.csv; rm -f gpurun_out/q7/exp.ncu-rep
