set -x
mkdir -p gpurun_out
TAG=${TAG:-r02q}
timeout 900 python -m pytest tests/test_gpu_tf32.py tests/test_gpu_shard.py tests/test_gpu_fullsize.py -m gpu -x -q -k "prune or shard or config4 or one_term or two_phase" > gpurun_out/pytest_band_$TAG.log 2>&1; echo "pytest rc $?"
tail -n 2 gpurun_out/pytest_band_$TAG.log
for b in 1 0; do
MC_BAND_WIDTH_SORT=$b timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench4_${TAG}_b$b.json 2> gpurun_out/bench4_${TAG}_b$b.err; echo "bench4 b$b rc $?"
done
timeout 900 ncu --set full --clock-control none -k regex:cv_grad_i8_kernel -c 1 -o gpurun_out/full_gi8_T131072_$TAG python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_gi8_full_$TAG.log 2>&1; echo "ncu rc $?"
echo done
