#!/bin/bash
# Streamed e2e input check (run via gpurun): the chunked-copy tests must pass, and must FAIL when
# the joins' chunk waits are compiled out (a copy of the tree; proves the poison test has teeth);
# then the C5 e2e timeline with MAPSQ_DEBUG.
OUT=gpurun_out/stream; mkdir -p $OUT
python build.py > $OUT/build.log 2>&1 || { echo build failed; exit 1; }
timeout 900 python -m pytest tests/test_gpu_index.py -x -q > $OUT/pytest.log 2>&1; echo "index tests rc=$?"; tail -2 $OUT/pytest.log
rm -rf /tmp/brk && mkdir /tmp/brk && cp -r . /tmp/brk/ 2>/dev/null
( cd /tmp/brk && sed -i '/^mapsq_status wait_stream_b(mapsq_ctx \*ctx, uint64_t rows, cudaStream_t s) {/a\  if (rows) return MAPSQ_OK;' paper_1702_03484_b200/csrc/api.cu && \
  grep -c "if (rows) return MAPSQ_OK" paper_1702_03484_b200/csrc/api.cu && \
  python build.py --force > /dev/null 2>&1 && \
  timeout 600 python -m pytest tests/test_gpu_index.py -x -q -k streamed > /root/repo/$OUT/pytest_broken.log 2>&1; echo "broken-wait tests rc=$? (must be 1)" )
tail -2 $OUT/pytest_broken.log
MAPSQ_DEBUG=1 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline 2> $OUT/debug.err > $OUT/bench_C5.json
grep "e2e ms" $OUT/debug.err | tail -2
python -c "import json; d=json.load(open('$OUT/bench_C5.json')); print(d['ms_per_step'], d['e2e'])"
