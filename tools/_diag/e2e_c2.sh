# config-2 e2e chunk schedules (compute-bound: fewer, larger chunks; small first/last)
for L in "list:4096,28672,28672,4096" "list:8192,49152,8192" "list:2048,30720,30720,2048" ""; do
  MC_E2E_CHUNKS="$L" python bench.py --config 2 --no-cpu --steps 3 --warmup 3 > gpurun_out/c2e.log 2>&1
  echo "[$L] $(tail -1 gpurun_out/c2e.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['e2e']['ms_per_step'], d['e2e']['value'], d['ms_per_step'])")"
done
