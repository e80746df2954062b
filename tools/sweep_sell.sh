#!/bin/bash
# unroll (RCG_SELL_U) x occupancy (RCG_SELL_MINB) x grid (RCG_SELL_CTAS) sweep of the sliced 3x3-block SpMV,
# beside the plain BSR and scalar CSR paths (libraries prebuilt under tools/_sv/)
for v in tools/_sv/librcg_sell_*.so; do for ct in 0 8 16; do
  echo -n "$(basename $v) ctas=$ct: "
  if [ $ct = 0 ]; then RCG_LIB=$v python tools/spmv_bench.py ${1:-elast64} bsr3; else RCG_LIB=$v RCG_SELL_CTAS=$ct python tools/spmv_bench.py ${1:-elast64} bsr3; fi
done; done
echo -n "plain bsr3: "; RCG_SELL=0 python tools/spmv_bench.py ${1:-elast64} bsr3
echo -n "csr: "; python tools/spmv_bench.py ${1:-elast64} csr
