# int8 gradient with wide groups (streamed A): tests, then config 3 bench
set -x
mkdir -p gpurun_out
TAG=${TAG:-r02c}
timeout 900 python -m pytest tests/test_gpu_grad_i8.py tests/test_gpu_parity.py -m gpu -x -q -k "i8 or close or config3" > gpurun_out/pytest_wide_$TAG.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/pytest_wide_$TAG.log
timeout 900 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench3_$TAG.json 2> gpurun_out/bench3_$TAG.err; echo "bench3 rc $?"
tail -3 gpurun_out/bench3_$TAG.err
echo done
