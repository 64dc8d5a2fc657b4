python build.py > /dev/null 2>&1 || exit 1
mkdir -p gpurun_out/q4
timeout 900 python -m pytest tests/test_gpu_semijoin.py tests/test_gpu_parity.py tests/test_gpu_index.py -x -q > gpurun_out/q4/pytest.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/q4/pytest.log
timeout 600 ncu --set full --import-source on -k regex:"filter" --launch-skip 2 --launch-count 2 -o gpurun_out/q4/filt -f python bench.py --config C4 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/q4/ncu.log 2>&1; echo "ncu rc=$?"
ncu -i gpurun_out/q4/filt.ncu-rep --page raw --csv > gpurun_out/q4/filt_raw.csv
for k in filter_build pack_filter; do ncu -i gpurun_out/q4/filt.ncu-rep --page source --csv --kernel-name regex:$k --launch-count 1 > gpurun_out/q4/src_$k.csv; done
gzip -f gpurun_out/q4/*.csv; rm -f gpurun_out/q4/filt.ncu-rep
