# in-solve A/B on config 3 (2 systems): tools/ab_config3_short.sh NAME...
for v in "$@"; do
  if [ "$v" = main ]; then unset RCG_LIB; else export RCG_LIB=$PWD/paper_1301_7530_b200/ab/$v/librcg.so; fi
  python bench.py --systems 2 --steps 2 --warmup 1 --no-cpu --no-e2e --no-secondary 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); r=d['roofline']
print('$v', round(d['value'],1), round(d['ms_per_step'],1), {k:(round(v['seconds'],4), round(v['GBps'])) for k,v in r['all_kernels'].items() if v['launches']}, d['clocks']['sm_mhz'])
"
done
