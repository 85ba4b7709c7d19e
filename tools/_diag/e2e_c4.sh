# config-4 e2e chunk schedules: geometric tapers (model-suggested) vs the default
for L in "list:8064,10624,10208,9824,9440,9088,8736,8416,8096,7776,7488,7200,6912,6656,6400,6144" "list:10688,15136,13952,12864,11840,10912,10048,9248,8512,7840,7232,6656,6144" "list:9152,17152,15808,14560,13408,12352,11392,10496,9664,8896,8192" ""; do
  MC_E2E_CHUNKS="$L" python bench.py --no-cpu --steps 4 --warmup 3 > gpurun_out/c4e.log 2>&1
  echo "[${L:0:30}] $(tail -1 gpurun_out/c4e.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['e2e']['ms_per_step'], d['e2e']['value'], d['ms_per_step'])")"
done
