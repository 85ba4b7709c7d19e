mkdir -p gpurun_out
TAG=${TAG:-r02aa}
timeout 900 python -m pytest tests/test_gpu_toysim.py -m gpu -x -q > gpurun_out/pytest_toy_$TAG.log 2>&1; echo "pytest rc $?"
tail -n 3 gpurun_out/pytest_toy_$TAG.log
