# timing of the int8 gradient kernel with stages switched off (MC_GI8_DBG, results invalid)
for d in ${DBGS:-0 16 144 272 400 146}; do
  MC_GI8_DBG=$d timeout 300 python bench.py --frames ${FRAMES:-16384} --steps 2 --warmup 1 --no-cpu 2>/dev/null | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read())
k = d['kernels']
print('dbg $d', 'grad_i8 %.2f ms' % k['mc_pathcv_grad_i8']['ms_per_step'], 'refine %.2f' % k.get('mc_refine', {}).get('ms_per_step', 0), 'step %.1f' % d['ms_per_step'])"
done
