# Round-2 measurement pass on one B200: the GPU test suite, smoke(), the default bench line
# (config 4, with the CPU baseline), the reference arm, and configs 0-3.
set -x
mkdir -p gpurun_out
TAG=${TAG:-r02final}
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc $?"
tail -n 3 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc $?"
tail -n 2 gpurun_out/smoke_$TAG.log
timeout 900 python bench.py > gpurun_out/bench4_$TAG.json 2> gpurun_out/bench4_$TAG.err; echo "bench4 rc $?"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref4_$TAG.json 2> gpurun_out/ref4_$TAG.err; echo "ref rc $?"
for c in 2 3 1 0; do
  timeout 900 python bench.py --config $c > gpurun_out/bench${c}_$TAG.json 2> gpurun_out/bench${c}_$TAG.err; echo "bench$c rc $?"
done
echo done
