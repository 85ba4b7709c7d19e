mkdir -p gpurun_out
TAG=${TAG:-r02x}
timeout 900 python bench.py --no-cpu > gpurun_out/bench4_$TAG.json 2> gpurun_out/bench4_$TAG.err; echo "bench4 rc $?"
timeout 600 python -m pytest tests/test_gpu_shard.py -m gpu -q -k two_phase > gpurun_out/pytest_2p_$TAG.log 2>&1; echo "pytest rc $?"
tail -n 1 gpurun_out/pytest_2p_$TAG.log
