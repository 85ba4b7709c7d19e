ncu --set full --clock-control none --import-source on -k regex:cv_grad_dmma -c 1 -o gpurun_out/grad_v18 python bench.py --frames 16384 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_g.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:refine_dmma -s 1 -c 1 -o gpurun_out/refine_v18 python bench.py --frames 16384 --steps 1 --warmup 1 --no-cpu > gpurun_out/ncu_r.log 2>&1
echo done
