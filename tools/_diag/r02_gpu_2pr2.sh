set -x
mkdir -p gpurun_out
TAG=${TAG:-r02s}
timeout 600 python -m pytest tests/test_gpu_shard.py -m gpu -x -q -k two_phase > gpurun_out/pytest_2pr2_$TAG.log 2>&1; echo "pytest rc $?"
tail -n 2 gpurun_out/pytest_2pr2_$TAG.log
timeout 600 python bench.py --shard landmarks --steps 3 --warmup 2 --no-cpu > gpurun_out/bench4_${TAG}_routed.json 2>&1; echo "bench rc $?"
timeout 1500 python tools/_diag/twophase_projection.py --routed 1 > gpurun_out/twophase_routed_$TAG.jsonl 2> gpurun_out/twophase_routed_$TAG.err; echo "proj rc $?"
tail -n 3 gpurun_out/twophase_routed_$TAG.err
echo done
