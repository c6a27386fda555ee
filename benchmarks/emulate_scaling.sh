# one B200 decodes every rank's shard of the 2-, 4- and 8-way snake split in turn (bench.py
# --emulate-shard R/W); the slowest rank of each W is the emulated N-GPU step time
out=gpurun_out/r02_emulated_shards.jsonl; : > $out
for W in 2 4 8; do for R in $(seq 0 $((W-1))); do
python bench.py --steps 3 --warmup 2 --no-cpu --no-configs --no-stamps --emulate-shard $R/$W 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print(json.dumps({'emulated_shard': d['emulated_shard'], 'value': round(d['value']), 'e2e': round(d['e2e']['value']), 'step_ms': [round(x,1) for x in d['step_ms']], 'batches_per_rank': d['config']['batches_per_rank']}))" >> $out
done; done
cat $out
