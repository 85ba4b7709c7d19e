EXPS="0 6 14 22 30 5" bash tools/_diag/r02_s4_gi8_exp.sh
