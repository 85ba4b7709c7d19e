mkdir -p gpurun_out
TAG=${TAG:-r02ab}
timeout 600 python -m pytest tests/test_gpu_grad_i8.py -m gpu -x -q -k "refit or digit" > gpurun_out/pytest_ri8b_$TAG.log 2>&1; echo "pytest rc $?"
tail -n 1 gpurun_out/pytest_ri8b_$TAG.log
timeout 900 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench2_$TAG.json 2>/dev/null; echo "bench2 rc $?"
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench4_$TAG.json 2>/dev/null; echo "bench4 rc $?"
