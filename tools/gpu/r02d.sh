set -x
./tools/k3lb 2709792 1000 > gpurun_out/r02d_k3lb.log 2>&1; echo k3lb rc=$?
cat gpurun_out/r02d_k3lb.log
timeout 900 python tools/run_configs.py 3 --systems 4 --no-rerun > gpurun_out/r02d_config3_4sys.json 2> gpurun_out/r02d_config3.err; echo c3 rc=$?
python -c "
import json; d=json.load(open('gpurun_out/r02d_config3_4sys.json')); print(d['iterations'], d['sequence_seconds_profiled'], d['kernels'])"
