#!/bin/bash
# unroll (RCG_SELL_U) x occupancy (RCG_SELL_MINB) sweep of the sliced 3x3-block SpMV, mode 0 (rcg_spmv)
# and the solve-loop kernel (RCG_SPMV_IND=1), beside plain BSR and scalar CSR (libraries prebuilt under tools/_sv/)
for v in tools/_sv/librcg_sell_*.so; do for ind in 0 1 2; do
  echo -n "$(basename $v) ind=$ind: "; RCG_LIB=$v RCG_SPMV_IND=$ind python tools/spmv_bench.py ${1:-elast64} bsr3
done; done
for ind in 0 1 2; do
echo -n "plain bsr3 ind=$ind: "; RCG_SPMV_IND=$ind RCG_SELL=0 python tools/spmv_bench.py ${1:-elast64} bsr3
echo -n "csr ind=$ind: "; RCG_SPMV_IND=$ind python tools/spmv_bench.py ${1:-elast64} csr
done
