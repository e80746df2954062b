./tools/k3lb 2709792 1000 2>&1 | head -9
for w in 1 2 3 4 6; do
  RCG_PRE_WAVES=$w timeout 600 python tools/run_configs.py 3 --systems 3 --no-rerun > gpurun_out/r02e_w$w.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/r02e_w$w.json')); k=d['kernels']; print('waves $w', d['iterations'], round(d['sequence_seconds_profiled'],3), 'precond', k['precond'], 'wupdate', k['wupdate'])"
done
