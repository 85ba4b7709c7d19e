# session-4 profile pass: launch list of one config-4 step, --set full captures of the int8
# gradient and refit kernels on a T = 16384 slice, the gradient at full size (DRAM traffic),
# and the refit kernel on a config-2 slice; each command first exits 0 without ncu.
set -x
mkdir -p gpurun_out
TAG=${TAG:-s4}
RE='regex:cv_grad|refine|msd_|center_split|rdig|gather|prune|cand|band|sort|cstack|weights|plan|ldig'
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/b_plain_$TAG.json 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$RE" -c 200 --csv \
  --log-file gpurun_out/launches4_$TAG.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launch rc $?"
timeout 300 python bench.py --frames 16384 --steps 1 --warmup 1 --no-cpu > gpurun_out/b_slice_$TAG.json 2>&1 || exit 1
for K in cv_grad_i8_kernel refine_i8_kernel; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -c 1 -o gpurun_out/full_${K}_$TAG \
    python bench.py --frames 16384 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_full_${K}_$TAG.log 2>&1; echo "ncu $K rc $?"
done
timeout 900 ncu --set full --clock-control none -k regex:cv_grad_i8_kernel -c 1 -o gpurun_out/full_gi8_T131072_$TAG \
  python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_full_gi8_T131072_$TAG.log 2>&1; echo "ncu full-size rc $?"
timeout 300 python bench.py --config 2 --frames 8192 --steps 1 --warmup 1 --no-cpu > gpurun_out/b_c2slice_$TAG.json 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:refine_i8_kernel -c 1 -o gpurun_out/full_refine_c2_$TAG \
  python bench.py --config 2 --frames 8192 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_full_refine_c2_$TAG.log 2>&1; echo "ncu c2 rc $?"
ls -la gpurun_out/*.ncu-rep
echo done
