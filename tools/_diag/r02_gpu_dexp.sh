set -x
mkdir -p gpurun_out
TAG=${TAG:-r02h}
timeout 900 python -m pytest tests/test_gpu_grad_i8.py tests/test_gpu_tf32.py tests/test_gpu_fullsize.py -m gpu -x -q -k "digit or i8 or uniform or config4 or config2 or split" > gpurun_out/pytest_dexp_$TAG.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/pytest_dexp_$TAG.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench4_$TAG.json 2> gpurun_out/bench4_$TAG.err; echo "bench4 rc $?"
timeout 900 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench2_$TAG.json 2> gpurun_out/bench2_$TAG.err; echo "bench2 rc $?"
echo done
