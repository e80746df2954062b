python -m pytest tests -m gpu -q > gpurun_out/r02s_gpu_tests.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/r02s_gpu_tests.log
