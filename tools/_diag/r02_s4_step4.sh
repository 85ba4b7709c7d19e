timeout 900 python -m pytest tests/test_gpu_grad_i8.py -x -q -m gpu 2>&1 | tail -3
EXPS="0 6 5" bash tools/_diag/r02_s4_gi8_exp.sh
export MCB200_LIB=$PWD/paper_1801_02362_b200/libmcb200_mmaexp.so
echo "== MMA issue experiments (no TMA, drain-only epilogue): 5 = all, +32 one N=192, +64 B as SW128, +128 four N=192"
EXPS="5 37 69 133" bash tools/_diag/r02_s4_gi8_exp.sh
