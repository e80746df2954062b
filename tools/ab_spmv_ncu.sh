# DRAM bytes of the solve-loop DIA SpMV per build (ncu, one launch): tools/ab_spmv_ncu.sh NELEM NAME...
export RCG_SPMV_IND=1 NELEM=$1; shift
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct"
for v in "$@"; do
  if [ "$v" = main ]; then unset RCG_LIB; else export RCG_LIB=$PWD/paper_1301_7530_b200/ab/$v/librcg.so; fi
  ncu --metrics $M --clock-control none -k regex:dia_kernel --launch-skip 10 --launch-count 1 --csv python tools/spmv_bench.py elast64 2>&1 \
    | grep "Command line" | awk -F'","' -v v=$v '{gsub(/"/,"",$NF); printf "[%s] %s %s\n", v, $(NF-2), $NF}'
done
