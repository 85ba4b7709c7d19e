mkdir -p gpurun_out
TAG=${TAG:-r02w}
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc $?"
tail -n 3 gpurun_out/pytest_gpu_$TAG.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc $?"
tail -n 1 gpurun_out/smoke_$TAG.log
