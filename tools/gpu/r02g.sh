python -m pytest tests -m gpu -x -q > gpurun_out/r02g_gpu_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/r02g_gpu_tests.log
timeout 600 python tools/run_configs.py 3 --systems 3 --no-rerun > gpurun_out/r02g_c3.json 2>/dev/null
python -c "
import json; d=json.load(open('gpurun_out/r02g_c3.json')); k=d['kernels']; print(d['iterations'], round(d['sequence_seconds_profiled'],3), 'precond', k['precond'], 'wupdate', k['wupdate'], 'spmv', k['spmv'])"
