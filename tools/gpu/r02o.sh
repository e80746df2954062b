python -m pytest tests/test_gpu_sequence_parity.py -q -x > gpurun_out/r02o_seq.log 2>&1; echo seq rc=$?
tail -15 gpurun_out/r02o_seq.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"precond_kernel|wupdate_kernel" --launch-skip 1980 --launch-count 2 -o gpurun_out/r02o_c3_k3k5 -f python tools/ncu_target.py 3 1000 > gpurun_out/r02o_ncu.log 2>&1; echo ncu rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02o_launches.csv python bench.py --steps 1 --warmup 0 --nelem 24 --systems 3 --no-cpu --no-secondary > gpurun_out/r02o_launch_bench.log 2>&1; echo launches rc=$?
