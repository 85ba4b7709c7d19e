mkdir -p gpurun_out
TAG=${TAG:-r02v}
timeout 600 python -m pytest tests/test_gpu_shard.py -m gpu -x -q -k two_phase > gpurun_out/pytest_2p3_$TAG.log 2>&1; echo "pytest rc $?"
tail -n 2 gpurun_out/pytest_2p3_$TAG.log
PROJ_KERNELS=1 timeout 1500 python tools/_diag/twophase_projection.py --routed 1 > gpurun_out/twophase_r1_$TAG.jsonl 2> gpurun_out/twophase_r1_$TAG.err; echo "proj rc $?"
