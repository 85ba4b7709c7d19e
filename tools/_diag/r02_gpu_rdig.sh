set -x
mkdir -p gpurun_out
TAG=${TAG:-r02n}
timeout 600 python -m pytest tests/test_gpu_grad_i8.py -m gpu -x -q -k "digit or refit" > gpurun_out/pytest_rdig_$TAG.log 2>&1; echo "pytest rc $?"
tail -n 2 gpurun_out/pytest_rdig_$TAG.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench4_$TAG.json 2> gpurun_out/bench4_$TAG.err; echo "bench4 rc $?"
echo done
