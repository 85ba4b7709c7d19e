# int8 gradient stage-removal diagnostics incl. bit 2 (no B boxes loaded); results invalid
for e in ${EXPS:-0 4 5 6 2 0}; do
  MC_GI8_EXP=$e timeout 300 python bench.py --frames 32768 --steps 3 --warmup 2 --no-cpu 2>/dev/null | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read())
k = d['kernels']
print('exp $e', {n: round(v['ms_per_step'], 2) for n, v in k.items() if 'grad' in n or 'refine' in n}, d['clocks']['sm_mhz'])"
done
