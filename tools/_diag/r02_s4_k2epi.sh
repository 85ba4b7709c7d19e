# one-term screen with 12 epilogue warps (diagnostic build -DMC_K2_EPI_WARPS=12) vs 8
for lib in libmcb200.so libmcb200_e12.so; do
  echo "== $lib"
  MCB200_LIB=$PWD/paper_1801_02362_b200/$lib timeout 600 python -m pytest tests/test_gpu_tf32.py -x -q -m gpu 2>&1 | tail -1
  MCB200_LIB=$PWD/paper_1801_02362_b200/$lib timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "
import json, sys
d = json.loads(sys.stdin.read())
print(round(d['ms_per_step'], 2), {k: round(v['ms_per_step'], 2) for k, v in d['kernels'].items() if 'msd' in k}, d['clocks']['sm_mhz'])"
done
