python tools/chol_bench.py 2>&1 | tail -8
RCG_CHOL_COLUMNS=1 python tools/chol_bench.py 2>&1 | tail -8
python -m pytest tests/test_gpu_kernels.py -q -x -k "cholesky" 2>&1 | tail -3
python -m pytest tests/test_gpu_sequence_parity.py -q -x -k "acceptance or trks" 2>&1 | tail -3
timeout 900 python bench.py --steps 3 --warmup 1 --no-cpu --no-secondary > gpurun_out/r02j_bench.log 2>&1; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r02j_bench.log').read().strip().splitlines()[-1]); print(d['value'], d['e2e'], d['roofline']['achieved'], d['roofline']['kernel'])"
