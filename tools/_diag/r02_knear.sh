for kn in 2 4 6 8; do
  MC_KNEAR=$kn timeout 300 python bench.py --steps 4 --warmup 2 --no-cpu 2>/dev/null | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read())
k = d['kernels']
print('knear $kn', round(d['ms_per_step'], 2), {n: round(v['ms_per_step'], 2) for n, v in k.items() if n in ('mc_msd_f16', 'mc_prune_plan', 'mc_gather_rows')}, d['config'].get('screen_tiles_computed_frac'), d['clocks']['sm_mhz'])"
done
