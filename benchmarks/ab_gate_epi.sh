set -x
B="python bench.py --steps 3 --warmup 3 --no-cpu --no-configs"
QNMT_GATE_EPI=0 $B > gpurun_out/ge_off.json 2>gpurun_out/ge_off.err
QNMT_GATE_EPI=1 $B > gpurun_out/ge_on.json 2>gpurun_out/ge_on.err
QNMT_GRU_BN=128,0 $B > gpurun_out/ge_128_0.json 2>/dev/null
QNMT_GRU_BN=128,64 $B > gpurun_out/ge_128_64.json 2>/dev/null
QNMT_GRU_BN=160,128 $B > gpurun_out/ge_160_128.json 2>/dev/null
QNMT_GRU_BN=192,96 $B > gpurun_out/ge_192_96.json 2>/dev/null
for f in ge_off ge_on ge_128_0 ge_128_64 ge_160_128 ge_192_96; do python -c "
import json,sys
d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', round(d['value']), round(d['e2e']['value']), d['ms_per_step'])"; done
