./tools/k3lb 2709792 1000 0 2>&1 | head -16
./tools/k3lb 2709792 1000 512 2>&1 | head -16
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"precond_kernel|wupdate_kernel" --launch-skip 1980 --launch-count 2 -o gpurun_out/r02f_c3_k3k5 -f python tools/ncu_target.py 3 1000 > gpurun_out/r02f_ncu.log 2>&1; echo ncu rc=$?
