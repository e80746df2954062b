python -m pytest tests -m gpu -x -q > gpurun_out/r02n_gpu_tests.log 2>&1; echo tests rc=$?
tail -3 gpurun_out/r02n_gpu_tests.log
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r02n_bench.log 2>&1; echo bench rc=$?
tail -c 600 gpurun_out/r02n_bench.log
