set -x
mkdir -p gpurun_out
TAG=${TAG:-r02o}
timeout 900 python -m pytest tests/test_gpu_grad_i8.py tests/test_gpu_parity.py -m gpu -x -q -k "i8 or close or config3 or force" > gpurun_out/pytest_gi8_$TAG.log 2>&1; echo "pytest rc $?"
tail -n 2 gpurun_out/pytest_gi8_$TAG.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench4_$TAG.json 2> gpurun_out/bench4_$TAG.err; echo "bench4 rc $?"
tail -n 3 gpurun_out/bench4_$TAG.err
echo done
