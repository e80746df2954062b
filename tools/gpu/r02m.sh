for v in B C E B C; do
  RCG_LIB=paper_1301_7530_b200/ab/$v/librcg.so timeout 180 python tools/run_configs.py 3 --systems 3 --no-rerun > gpurun_out/r02m_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/r02m_$v.json')); k=d['kernels']; print('$v', d['iterations'], round(d['sequence_seconds_profiled'],3), 'precond', k['precond'], 'wupdate', k['wupdate'])" 2>/dev/null || echo "$v failed"
done
