# config-4 bench with the D2H-first e2e schedule, then the launch list and ncu captures
set -x
mkdir -p gpurun_out
TAG=${TAG:-r02p}
timeout 900 python bench.py --no-cpu > gpurun_out/bench4_$TAG.json 2> gpurun_out/bench4_$TAG.err; echo "bench4 rc $?"
KERNELS="cv_grad_i8_kernel refine_i8_kernel msd_tf32_kernel center_split_f16x1_uni rdig_kernel" TAG=$TAG bash tools/_diag/r02_prof.sh
echo done
