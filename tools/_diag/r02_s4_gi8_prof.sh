# clock64 accounting of the int8 gradient kernel (diagnostic build -DMC_GI8_PROF)
for e in ${EXPS:-0 5 6}; do  # needs: python paper_1801_02362_b200/build.py -DMC_GI8_PROF --out=$PWD/paper_1801_02362_b200/libmcb200_prof.so
  echo "== exp $e"
  MCB200_LIB=$PWD/paper_1801_02362_b200/libmcb200_prof.so MC_GI8_EXP=$e timeout 300 python bench.py --frames 32768 --steps 1 --warmup 1 --no-cpu 2>&1 | grep gi8prof | tail -4
done
