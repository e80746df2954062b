# The sharded iteration (halo pack -> ncclSend/ncclRecv to self -> unpack, slab SpMV, 3 packed allreduces, captured
# in the batch graphs) against the plain path on ONE GPU: config 3 (96^3), 2 systems, two virtual slabs.
#   bash tools/shard_one_bench.sh [NELEM=96]
NE=${1:-96}
pick='import json,sys
d=json.loads([l for l in sys.stdin.read().splitlines() if l.startswith("{")][-1]); r=d["roofline"]
print(round(d["value"],1), "iters/s", round(d["ms_per_step"],1), "ms/step", d["config"]["parallelism"], d["phases_profiled_step"], {k:(round(v["seconds"],4), round(v["GBps"])) for k,v in r["all_kernels"].items() if v["launches"]})'
echo "plain:"; python bench.py --nelem $NE --systems 2 --steps 2 --warmup 3 --no-cpu --no-e2e --no-secondary 2>&1 | python -c "$pick"
for ov in 1 0; do
  echo "sharded (virtual slabs, NCCL self exchange), RCG_HALO_OVERLAP=$ov:"
  RCG_HALO_OVERLAP=$ov RCG_COMM_FORCE=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 2952$ov \
    bench.py --gpus 1 --shard-one --nelem $NE --systems 2 --steps 2 --warmup 3 --no-cpu --no-e2e 2>&1 | python -c "$pick"
done
