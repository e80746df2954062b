#!/bin/bash
# occupancy (RCG_SPMV_MINB variants) x grid (RCG_BSR_CTAS) sweep of the 3x3-block SpMV
for mb in 2 3 4 5; do for ct in 4 8 16; do
  echo -n "minb=$mb ctas=$ct: "
  RCG_LIB=tools/_var/librcg_mb$mb.so RCG_BSR_CTAS=$ct python tools/spmv_bench.py elast64 bsr3
done; done
for mb in 2 3 4 5; do echo -n "csr minb=$mb: "; RCG_LIB=tools/_var/librcg_mb$mb.so python tools/spmv_bench.py elast64 csr; done
