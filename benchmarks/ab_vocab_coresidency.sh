B="python bench.py --steps 3 --warmup 3 --no-cpu --no-configs"
L=paper_1804_05038_b200/_lib
python -m pytest tests/test_gpu_vocab_shard.py -x -q 2>&1 | tail -2
for v in "" _vt3 _vt3r104 _vt3r96; do
QNMT_LIB_PATH=$PWD/$L/libqnmt_b200$v.so $B 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']; print('variant[$v]', round(d['value']), round(d['e2e']['value']), 'vocab_stats us', round(k['vocab_stats']['us_per_launch'],1), 'att us', round(k['attention']['us_per_launch'],1))"
done
