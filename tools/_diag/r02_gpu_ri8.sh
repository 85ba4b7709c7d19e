set -x
mkdir -p gpurun_out
TAG=${TAG:-r02i}
timeout 900 python -m pytest tests/test_gpu_grad_i8.py -m gpu -x -q -k "refit" > gpurun_out/pytest_ri8_$TAG.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/pytest_ri8_$TAG.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench4_$TAG.json 2> gpurun_out/bench4_$TAG.err; echo "bench4 rc $?"
timeout 900 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench2_$TAG.json 2> gpurun_out/bench2_$TAG.err; echo "bench2 rc $?"
echo done
