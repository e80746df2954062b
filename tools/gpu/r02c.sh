set -x
python -m pytest tests/test_gpu_sequence_parity.py tests/test_gpu_reference_bridge.py -q > gpurun_out/r02c_tests.log 2>&1; echo tests rc=$?
tail -30 gpurun_out/r02c_tests.log
# K3 / K5 at j ~ 990 of config 3 system 0 (launch 0 of each is the init launch)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"precond_kernel|wupdate_kernel" --launch-skip 1980 --launch-count 2 -o gpurun_out/r02c_c3_k3k5 -f python tools/ncu_target.py 3 1000 > gpurun_out/r02c_ncu.log 2>&1; echo ncu rc=$?
tail -5 gpurun_out/r02c_ncu.log
