for v in B0 H1 B0 H1; do
  RCG_LIB=paper_1301_7530_b200/ab/$v/librcg.so timeout 300 python tools/run_configs.py 3 --systems 2 --no-rerun > gpurun_out/r02t_c3_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/r02t_c3_$v.json')); k=d['kernels']; print('c3 $v', d['iterations'], round(d['sequence_seconds_profiled'],3), 'spmv', k['spmv'])" 2>/dev/null || echo "$v failed"
  RCG_LIB=paper_1301_7530_b200/ab/$v/librcg.so timeout 300 python tools/run_configs.py 4 --systems 3 --reorth 0 --cap 400 --no-rerun > gpurun_out/r02t_c4_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/r02t_c4_$v.json')); k=d['kernels']; print('c4 $v', d['iterations'], round(d['sequence_seconds_profiled'],3), 'spmv', k['spmv'])" 2>/dev/null || echo "$v c4 failed"
done
