timeout 1500 python -m pytest tests/test_gpu_grad_i8.py tests/test_gpu_tf32.py -x -q -m gpu 2>&1 | tail -3
for c in 4 3; do
  timeout 900 python bench.py --config $c --no-cpu 2>/dev/null | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read())
print('config $c', round(d['value']), 'ms/step', round(d['ms_per_step'], 2), {k: round(v['ms_per_step'], 2) for k, v in d['kernels'].items() if v['ms_per_step'] > 0.3}, d['clocks']['sm_mhz'])"
done
