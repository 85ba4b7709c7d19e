# K1s (one-term F16 frame split) CTA size sweep on the config-4 shape (T = 32768)
for cfg in "MC_K1_NT=128" "MC_K1_NT=256" "MC_K1_NT=512"; do
  env $cfg python bench.py --frames 32768 --steps 3 --warmup 3 --no-cpu > gpurun_out/sw.log 2>&1
  echo "$cfg $(tail -1 gpurun_out/sw.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['kernels']['mc_center_split16'])")"
done
