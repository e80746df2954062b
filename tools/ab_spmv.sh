# A/B of the solve-loop DIA SpMV across librcg.so builds: tools/ab_spmv.sh NAME...
# ("main" = the in-tree build, others = paper_1301_7530_b200/ab/NAME/librcg.so)
export RCG_SPMV_IND=1
for v in "$@"; do
  if [ "$v" = main ]; then unset RCG_LIB; else export RCG_LIB=$PWD/paper_1301_7530_b200/ab/$v/librcg.so; fi
  for rep in 1 2; do
    echo "[$v] $(python tools/spmv_bench.py elast64 2>&1 | tail -1)"
    echo "[$v] $(NELEM=96 python tools/spmv_bench.py elast64 2>&1 | tail -1)"
    echo "[$v] $(python tools/spmv_bench.py diff256 2>&1 | tail -1)"
  done
done
