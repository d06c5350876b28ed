# round-2 batch 6: schedule variants of the pair kernels (local-leg cost),
# 4- and 8-rank torchrun benches with every rank on device 0 (validation)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2b6; mkdir -p $O
for d in 0 4 8; do
  MGG_AGG_DYN=$d timeout 600 python tools/hiding_b200.py --forms 1,4 --far 0.002,0.01 --out $O/loc_dyn$d.jsonl > /dev/null 2>&1
  MGG_AGG_DYN=$d timeout 300 python tools/hiding_b200.py --graph products-gcn --device-peer --forms 1,4 --reps 3 --out $O/dev_products_dyn$d.jsonl > /dev/null 2>&1
done
for n in 4 8; do
  MGG_BENCH_DEVICE=0 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n bench.py --gpus $n --steps 3 --warmup 3 --secondary none --no-cpu > $O/bench_${n}rank_1dev.json 2> $O/bench_${n}rank_1dev.err
  echo "n=$n rc=$?"; tail -c 300 $O/bench_${n}rank_1dev.json; grep -i error $O/bench_${n}rank_1dev.err | head -3
done
