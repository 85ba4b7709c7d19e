# pruned close-structure replay: parity tests, config-3 and config-2 bench lines
set -x
mkdir -p gpurun_out
TAG=${TAG:-r02b}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "close or config3 or eps_zero" > gpurun_out/pytest_c3_$TAG.log 2>&1; echo "pytest rc $?"
tail -5 gpurun_out/pytest_c3_$TAG.log
timeout 900 python bench.py --config 3 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench3_$TAG.json 2> gpurun_out/bench3_$TAG.err; echo "bench3 rc $?"
tail -3 gpurun_out/bench3_$TAG.err
timeout 600 python bench.py --config 2 --no-cpu > gpurun_out/bench2_$TAG.json 2> gpurun_out/bench2_$TAG.err; echo "bench2 rc $?"
tail -3 gpurun_out/bench2_$TAG.err
echo done
