# Launch list of the library's kernels over one timed config-4 step (ncu, cold-cache,
# serialised: shares, not absolutes) and --set full captures of the top kernels on a
# T = 16384 slice; each command first exits 0 without ncu.
set -x
mkdir -p gpurun_out
TAG=${TAG:-r02k}
RE='regex:cv_grad|refine|msd_|center_split|rdig|gather|prune|cand|band|sort|cstack|weights|plan|ldig'
timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/b_plain_$TAG.json 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k "$RE" -c 200 --csv \
  --log-file gpurun_out/launches4_$TAG.csv python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launch rc $?"
timeout 300 python bench.py --frames 16384 --steps 1 --warmup 1 --no-cpu > gpurun_out/b_slice_$TAG.json 2>&1 || exit 1
for K in ${KERNELS:-cv_grad_i8_kernel refine_i8_kernel cstack_prep}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -c 1 -o gpurun_out/full_${K}_$TAG \
    python bench.py --frames 16384 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_full_${K}_$TAG.log 2>&1; echo "ncu $K rc $?"
done
echo done
