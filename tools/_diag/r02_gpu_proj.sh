mkdir -p gpurun_out
TAG=${TAG:-r02t}
for r in 0 1; do
timeout 1500 python tools/_diag/twophase_projection.py --routed $r > gpurun_out/twophase_r${r}_$TAG.jsonl 2> gpurun_out/twophase_r${r}_$TAG.err; echo "proj $r rc $?"
done
