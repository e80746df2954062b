for t in 4 2 3 6 8 4; do
  echo -n "UPD_TILES=$t: "
  RCG_UPD_TILES_PER_SM=$t timeout 200 python bench.py --systems 2 --steps 1 --warmup 1 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['all_kernels']; print(round(d['value'],1), d['iterations_per_system'], {n:(round(v['seconds'],4), round(v['GBps'])) for n,v in k.items() if n in ('update','actr','spmv')})"
done
