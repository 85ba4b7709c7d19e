set -x
mkdir -p gpurun_out
TAG=${TAG:-r02r}
timeout 900 python -m pytest tests/test_gpu_shard.py -m gpu -x -q > gpurun_out/pytest_2pr_$TAG.log 2>&1; echo "pytest rc $?"
tail -n 2 gpurun_out/pytest_2pr_$TAG.log
for sh in landmarks landmarks-allgather; do
timeout 900 python bench.py --shard $sh --steps 3 --warmup 2 --no-cpu > gpurun_out/bench4_${TAG}_$sh.json 2> gpurun_out/bench4_${TAG}_$sh.err; echo "bench $sh rc $?"
tail -n 2 gpurun_out/bench4_${TAG}_$sh.err
done
echo done
