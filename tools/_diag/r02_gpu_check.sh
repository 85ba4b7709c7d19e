# Round-2 re-entry check on one B200: GPU tests, config-4 and config-2 bench lines,
# the config-4 launch list, and one ncu --set full capture each of the two int8
# tensor-core kernels (refits, gradient) on a T = 16384 slice.
set -x
mkdir -p gpurun_out
TAG=${TAG:-r02a}
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py > gpurun_out/bench4_$TAG.json 2> gpurun_out/bench4_$TAG.err; echo "bench4 rc $?"
timeout 600 python bench.py --config 2 --no-cpu > gpurun_out/bench2_$TAG.json 2> gpurun_out/bench2_$TAG.err; echo "bench2 rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches4_$TAG.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch_$TAG.log 2>&1; echo "launch rc $?"
for K in cv_grad_i8 refine_i8; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -c 1 -o gpurun_out/full_${K}_$TAG \
    python bench.py --frames 16384 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_full_${K}_$TAG.log 2>&1; echo "ncu $K rc $?"
done
echo done
