timeout 600 ncu --set full --clock-control none -k regex:"wu3|pre" --launch-skip 0 --launch-count 40 -o gpurun_out/r02i_k3lb -f ./tools/k3lb 2709792 1000 512 > gpurun_out/r02i_ncu_lb.log 2>&1; echo ncu1 rc=$?
timeout 600 python tools/e2e_upload.py > gpurun_out/r02i_e2e_upload.log 2>&1; echo e2e rc=$?
cat gpurun_out/r02i_e2e_upload.log
