export RCG_SPMV_IND=1
M="dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct,l1tex__t_sector_hit_rate.pct,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed,launch__registers_per_thread,launch__grid_size,smsp__inst_executed.sum"
for ne in 64 96; do
echo "== csr NELEM=$ne"; NELEM=$ne python tools/spmv_bench.py elast64 csr | tail -1
NELEM=$ne ncu --metrics $M --clock-control none -k regex:spmv_kernel --launch-skip 10 --launch-count 1 --csv python tools/spmv_bench.py elast64 csr 2>&1 | grep "Command line" | awk -F'","' '{gsub(/"/,"",$NF); printf "%s %s\n", $(NF-2), $NF}'
echo "== sell NELEM=$ne"; RCG_DIA=0 NELEM=$ne python tools/spmv_bench.py elast64 | tail -1
RCG_DIA=0 NELEM=$ne ncu --metrics $M --clock-control none -k regex:sell3_kernel --launch-skip 10 --launch-count 1 --csv python tools/spmv_bench.py elast64 2>&1 | grep "Command line" | awk -F'","' '{gsub(/"/,"",$NF); printf "%s %s\n", $(NF-2), $NF}'
done
