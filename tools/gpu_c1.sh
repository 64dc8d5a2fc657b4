#!/bin/bash
# C1 breakdown: host vs device time of the query call, plus an ncu capture of the one-launch small join
python build.py > /dev/null 2>&1
mkdir -p gpurun_out/c1
python tools/c1_breakdown.py 2>&1 | tail -3
ncu --set full --clock-control none --import-source on -k regex:small_join --launch-count 3 -o gpurun_out/c1/small -f python bench.py --config C1 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/c1/ncu.log 2>&1
ncu -i gpurun_out/c1/small.ncu-rep --page source --csv --launch-count 1 > gpurun_out/c1/source.csv 2>/dev/null
ncu -i gpurun_out/c1/small.ncu-rep --page details --csv > gpurun_out/c1/details.csv 2>/dev/null
rm -f gpurun_out/c1/small.ncu-rep
