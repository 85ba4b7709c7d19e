set -x
mkdir -p gpurun_out
TAG=${TAG:-r02g}
true
tail -3 gpurun_out/pytest_2p_$TAG.log
timeout 1200 python tools/_diag/twophase_projection.py > gpurun_out/twophase_$TAG.jsonl 2> gpurun_out/twophase_$TAG.err; echo "proj rc $?"
tail -3 gpurun_out/twophase_$TAG.err
echo done
