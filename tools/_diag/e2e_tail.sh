# e2e chunk schedule: size of the last (exposed) chunk, T / MC_E2E_TAIL
for d in 16 32 64; do
  MC_E2E_TAIL=$d python bench.py --no-cpu --steps 4 --warmup 3 > gpurun_out/e2e_$d.log 2>&1
  echo "tail T/$d $(tail -1 gpurun_out/e2e_$d.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['e2e']['ms_per_step'], d['e2e']['value'], d['ms_per_step'])")"
done
