mkdir -p gpurun_out
TAG=${TAG:-r02u}
for r in 0 1; do
PROJ_KERNELS=1 timeout 1500 python tools/_diag/twophase_projection.py --routed $r --gpus 1,2,4,8 > gpurun_out/twophase_r${r}_$TAG.jsonl 2> gpurun_out/twophase_r${r}_$TAG.err; echo "proj $r rc $?"
done
