python -m pytest tests/test_gpu_kernels.py -q -x -k "pinned" 2>&1 | tail -2
timeout 600 python tools/e2e_upload.py 2>&1 | tail -9
