# ncu of the int8 gradient kernel on a config-4 slice (T = 16384): launch times of the
# int8 kernel vs its DMMA fallback, then one --set full capture of cv_grad_i8_kernel
set -x
TAG=${TAG:-i8}
python bench.py --frames 16384 --steps 1 --warmup 1 --no-cpu > gpurun_out/b_plain_$TAG.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"cv_grad" -c 8 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --frames 16384 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_launch_$TAG.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"cv_grad_i8" -c 1 -o gpurun_out/full_$TAG python bench.py --frames 16384 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_full_$TAG.log 2>&1
echo done
