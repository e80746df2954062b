#!/bin/bash
# per-kernel-class live timing (bench roofline pass) for 2 systems of config 2 under env variants:
#   bash tools/kclass.sh "RCG_ACTR_CTAS_PER_SM=4" "RCG_ACTR_CTAS_PER_SM=16"
for v in "$@"; do
  env $v python bench.py --systems 2 --steps 1 --warmup 1 --no-e2e --no-cpu 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); r=d['roofline']
print('$v', round(d['ms_per_step'],1), 'ms', ' '.join(f\"{k}={v['seconds']*1e3:.1f}ms/{v['GBps']:.0f}\" for k,v in r['all_kernels'].items() if v['launches']))"
done
