# A/B a compile-time flag of libmapsq: bench C5 and C4 built with FLAG_B (env) vs the default
# build.  usage: FLAG_B="-DMAPSQ_L2_HINT=0" bash tools/ab_flag.sh
mkdir -p gpurun_out/ab; rm -f gpurun_out/ab/*
run() {
  for c in C5 C4 C5 C4; do
    timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['config']['workload'], round(d['ms_per_step'],3), {k:round(v['avg_ms']*v['launches']/d['steps'],3) for k,v in d['kernels'].items() if 'filter' in k})"
  done
}
python build.py --force > /dev/null 2>&1 || exit 1
run default
NVCC_APPEND_FLAGS="$FLAG_B" python build.py --force > /dev/null 2>&1 || exit 1
run B
