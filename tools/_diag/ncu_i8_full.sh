# one ncu --set full capture of cv_grad_i8_kernel at full config 4 (after a plain run)
set -x
TAG=${TAG:-i8v2}
python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/b_plain_$TAG.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"cv_grad_i8" -c 1 -o gpurun_out/full_$TAG python bench.py --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_full_$TAG.log 2>&1
echo done
