# int8 gradient with the epilogue math switched off (MC_GI8_EXP=1; results invalid) vs on
for e in ${EXPS:-0 1 3}; do
  MC_GI8_EXP=$e timeout 300 python bench.py --frames 32768 --steps 3 --warmup 2 --no-cpu 2>/dev/null | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read())
k = d['kernels']
print('exp $e', {n: round(v['ms_per_step'], 2) for n, v in k.items() if 'grad' in n or 'refine' in n}, d['clocks']['sm_mhz'])"
done
