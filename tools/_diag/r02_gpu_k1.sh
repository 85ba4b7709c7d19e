# uniform K1s: tests, config-4 bench
set -x
mkdir -p gpurun_out
TAG=${TAG:-r02d}
timeout 900 python -m pytest tests/test_gpu_tf32.py tests/test_gpu_grad_i8.py tests/test_gpu_fullsize.py -m gpu -x -q -k "split or one_term or prune or config4 or i8" > gpurun_out/pytest_k1_$TAG.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/pytest_k1_$TAG.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench4_$TAG.json 2> gpurun_out/bench4_$TAG.err; echo "bench4 rc $?"
tail -3 gpurun_out/bench4_$TAG.err
echo done
