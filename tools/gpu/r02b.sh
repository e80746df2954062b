set -x
python -m pytest tests/test_gpu_sequence_parity.py -x -q -k "not c4r and not c5r and not config2_full" > gpurun_out/r02b_seq_tests.log 2>&1; echo seqtests rc=$?
tail -5 gpurun_out/r02b_seq_tests.log
timeout 300 python bench.py --nelem 16 --systems 5 --steps 3 --warmup 2 --cpu-iters 5 > gpurun_out/r02b_bench_small.log 2>&1; echo small rc=$?
tail -c 1500 gpurun_out/r02b_bench_small.log
timeout 1500 python bench.py --steps 4 --warmup 2 > gpurun_out/r02b_bench.log 2>&1; echo bench rc=$?
tail -c 3000 gpurun_out/r02b_bench.log
