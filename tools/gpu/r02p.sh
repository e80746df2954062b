python -m pytest tests/test_gpu_sequence_parity.py -q > gpurun_out/r02p_seq.log 2>&1; echo seq rc=$?
tail -5 gpurun_out/r02p_seq.log
