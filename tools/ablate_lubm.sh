# digit-pass ablation on real join words (C5 at LUBM(2000)) and the C4-shaped Zipf sort; run via gpurun
mkdir -p gpurun_out/q2
python build.py > gpurun_out/q2/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_index.py -x -q 2>&1 | tail -3
timeout 600 python tools/dump_words.py C5 2000 /tmp/c5w 2>&1 | tail -3
for j in 1 2; do
  read -r _ path ib kb rest <<< "$(grep "^J$j" <(python -c "
import json; [print('J%d'%m['join'], m['path'], m['ib'], m['kb']) for m in json.load(open('/tmp/c5w_meta.json'))]"))"
  timeout 600 tools/radix_ablate file $path $ib $kb
done
timeout 900 tools/radix_ablate zipf 400000000
