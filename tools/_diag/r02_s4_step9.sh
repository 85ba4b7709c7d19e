timeout 900 python -m pytest tests/test_gpu_grad_i8.py -x -q -m gpu 2>&1 | tail -3
EXPS="0 6 5" bash tools/_diag/r02_s4_gi8_exp.sh
