# multi-process forward as a CUDA graph: two-process tests (x10), 2/4-rank benches on one device
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2mp; mkdir -p $O
timeout 1800 tools/ipc_loop.sh 10 $O/ipc_loop.txt > /dev/null 2>&1; tail -2 $O/ipc_loop.txt
for n in 2 4; do
  MGG_BENCH_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2955$n bench.py --gpus $n --steps 10 --warmup 3 --secondary none --no-cpu > $O/bench_${n}rank_1dev.json 2> $O/bench_${n}rank_1dev.err
  echo "n=$n rc=$?"; python -c "import json;r=json.loads(open('$O/bench_${n}rank_1dev.json').read().strip().splitlines()[-1]);print(r['ms_per_step'], r['value'], r['gpu_launches'], r['e2e']['value'])"; grep -i "error" $O/bench_${n}rank_1dev.err | head -3
done
