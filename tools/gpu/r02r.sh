RCG_PARITY_DUMP=gpurun_out/r02r_c2_alone.json python -m pytest tests/test_gpu_sequence_parity.py -q -k config2 > gpurun_out/r02r_alone.log 2>&1; echo alone rc=$?
RCG_PARITY_DUMP=gpurun_out/r02r_c2_suite.json python -m pytest tests -m gpu -q -x --ignore=tests/test_gpu_sharded_loopback.py --ignore=tests/test_gpu_solver.py -k "not reduced and not benchmark and not acceptance and not trks and not cluster" > gpurun_out/r02r_suite.log 2>&1; echo suite rc=$?
tail -3 gpurun_out/r02r_suite.log
