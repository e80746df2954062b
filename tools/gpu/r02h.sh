./tools/k3lb 2709792 1000 512 2>&1 | tail -12
