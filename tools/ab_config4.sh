# config 4 (7-point 256^3, reorth off, krylov_cap 400), 2 systems: tools/ab_config4.sh NAME...
for v in "$@"; do
  if [ "$v" = main ]; then unset RCG_LIB; else export RCG_LIB=$PWD/paper_1301_7530_b200/ab/$v/librcg.so; fi
  python tools/run_configs.py 4 --systems 2 --reorth 0 --cap 400 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$v', d['iterations'], round(d['sequence_seconds'],3), round(d['iters_per_s']), d['kernels'])
"
done
