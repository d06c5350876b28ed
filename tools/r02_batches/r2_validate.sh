# round-2 validation batch (see DESIGN §5/§7): full GPU suite, the two-process
# IPC loop, hiding on the bench graphs, ablation, bench, 2-rank torchrun
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -4 > gpurun_out/r2_gputest.txt
cat gpurun_out/r2_gputest.txt
timeout 600 python bench.py > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err
tail -c 300 gpurun_out/r2_bench.json
MGG_BENCH_DEVICE=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --secondary none > gpurun_out/r2_bench_2rank.json 2> gpurun_out/r2_bench_2rank.err
tail -c 400 gpurun_out/r2_bench_2rank.json
for gw in config1 products-gcn reddit-gcn; do
  timeout 600 python tools/hiding_b200.py --graph $gw --forms 1,2,0 --reps 3 --ps 16 --dist 8 --wpb 8 --out gpurun_out/r2_hiding_$gw.jsonl > /dev/null 2>&1
done
timeout 1200 python tools/ablation_b200.py --out gpurun_out/r2_ablation.jsonl > /dev/null 2>&1
timeout 1800 tools/ipc_loop.sh 50 gpurun_out/r2_ipc_loop.txt > /dev/null 2>&1
tail -3 gpurun_out/r2_ipc_loop.txt
