set -x
mkdir -p gpurun_out
TAG=${TAG:-r02l}
timeout 600 python -m pytest tests/test_gpu_grad_i8.py -m gpu -x -q -k "refit or digit" > gpurun_out/pytest_pair_$TAG.log 2>&1; echo "pytest rc $?"
tail -3 gpurun_out/pytest_pair_$TAG.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_tf32.py tests/test_neighbour.py -m gpu -x -q -k "close or config2 or exact or dense or neighbour or prune" > gpurun_out/pytest_pair2_$TAG.log 2>&1; echo "pytest2 rc $?"
tail -3 gpurun_out/pytest_pair2_$TAG.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/bench4_$TAG.json 2> gpurun_out/bench4_$TAG.err; echo "bench4 rc $?"
timeout 900 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/bench2_$TAG.json 2> gpurun_out/bench2_$TAG.err; echo "bench2 rc $?"
echo done
