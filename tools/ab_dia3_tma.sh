# A/B of the TMA-staged 3x3 block-DIA SpMV (RCG_DIA3_TMA) on the config-2 bench, 2 systems
export RCG_DIA3_TMA=1
timeout 300 python -m pytest tests -m gpu -x -q -k "dia or spmv or reference_suite or full_size or edge" > gpurun_out/tma_tests.log 2>&1; echo rc=$? >> gpurun_out/tma_tests.log
for cfg in "0 4" "1 4" "1 5" "1 6" "1 3" "0 4" "1 4"; do
  set -- $cfg
  echo -n "TMA=$1 S=$2: " >> gpurun_out/tma_ab.log
  RCG_DIA3_TMA=$1 RCG_DIA3T_S=$2 timeout 200 python bench.py --systems 2 --steps 1 --warmup 1 --no-cpu --no-e2e 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline']['all_kernels']; print(round(d['value'],1), {n:(round(v['seconds'],4), round(v['GBps'])) for n,v in k.items() if v['launches']})" >> gpurun_out/tma_ab.log 2>&1
done
