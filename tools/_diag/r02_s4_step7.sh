echo base; EXPS="0 6" bash tools/_diag/r02_s4_gi8_exp.sh
echo setmaxnreg; MCB200_LIB=$PWD/paper_1801_02362_b200/libmcb200_va.so EXPS="0 6" bash tools/_diag/r02_s4_gi8_exp.sh
echo tiletoken; MCB200_LIB=$PWD/paper_1801_02362_b200/libmcb200_vb.so EXPS="0 6" bash tools/_diag/r02_s4_gi8_exp.sh
