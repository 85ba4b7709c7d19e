set -x
mkdir -p gpurun_out
TAG=${TAG:-r02e}
timeout 900 python -m pytest tests/test_neighbour.py tests/test_gpu_tf32.py -m gpu -x -q -k "neighbour or uniform" > gpurun_out/pytest_nl_$TAG.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/pytest_nl_$TAG.log
echo done
