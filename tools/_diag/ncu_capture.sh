set -x
python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/b_plain.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_v18.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"cv_grad_dmma|refine_dmma|msd_tf32_kernel|center_split_f16x1" -c 4 -o gpurun_out/full_v18 python bench.py --frames 16384 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_full.log 2>&1
echo done
