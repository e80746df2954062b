for v in CSR0 CUR CSR0 CUR; do
  for V in 8 4; do
    RCG_SPMV_V=$V RCG_LIB=paper_1301_7530_b200/ab/$v/librcg.so python tools/spmv_bench.py elast64 csr 2>&1 | sed "s/^/$v /"
  done
  RCG_LIB=paper_1301_7530_b200/ab/$v/librcg.so python tools/spmv_bench.py elast64 csr 2>&1 | sed "s/^/$v auto-V /"
done
