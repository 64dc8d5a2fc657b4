#!/bin/bash
# CUB calibration of the radix sort (tools/cub_calibrate.cu, test-only) on J1- and C4-shaped words
OUT=gpurun_out/${TAG:-calib}; mkdir -p $OUT
python build.py > $OUT/build.log 2>&1 || exit 1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include tools/cub_calibrate.cu -o tools/cub_calibrate \
  -Lpaper_1702_03484_b200 -lmapsq -Xlinker -rpath='$ORIGIN/../paper_1702_03484_b200' > $OUT/nvcc.log 2>&1 || { tail $OUT/nvcc.log; exit 1; }
for args in "63000000 29 0" "70000000 29 0.1" "400000000 29 0" "1000000000 29 0.1"; do
  timeout 300 tools/cub_calibrate $args | tee -a $OUT/calib.jsonl
done
