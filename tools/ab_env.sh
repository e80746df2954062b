#!/bin/bash
# A/B env settings on one config-2 run (2 systems); prints value and per-kernel (s, GB/s)
# usage: tools/ab_env.sh "RCG_WU_RPT=4" "RCG_WU_RPT=8" ...
for v in "$@"; do
  echo -n "$v: "
  env $v timeout 300 python bench.py --systems ${AB_SYSTEMS:-2} --steps ${AB_STEPS:-1} --warmup 3 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['all_kernels']; print(round(d['value'],1), {n:(round(v['seconds'],3), round(v['GBps'])) for n,v in k.items() if v['launches']})"
done
