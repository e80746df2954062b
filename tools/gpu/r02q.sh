python tools/determinism_check.py 3
python tools/determinism_check.py 2
python -m pytest tests/test_gpu_kernels.py -q -x > /dev/null 2>&1; echo kernels-first
