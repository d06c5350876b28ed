# round-2 batch 4: K1 fetch-size sweep (+ ncu DRAM bytes), ncu of the pair
# kernel against a host-mapped peer, 2-rank torchrun bench on one device
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2b4; mkdir -p $O
timeout 900 python tools/k1_fetch_sweep.py --workloads products-gcn,orkut-gcn,orkut-rmat-gcn > $O/fetch_sweep.jsonl 2> $O/fetch_sweep.err
cat $O/fetch_sweep.jsonl | cut -c1-300
timeout 1200 bash tools/k1_fetch_ncu.sh $O/fetch_ncu.csv > /dev/null 2>&1
# pair kernel, host-mapped peer, rf 0.1%: every gpair launch with key metrics
MGG_AGG_PAIR=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:agg_ --csv --log-file $O/pair_hostpeer_metrics.csv python tools/hiding_b200.py --child --forms 1 --far 0.002 --reps 2 > $O/pair_hostpeer.log 2>&1
tail -2 $O/pair_hostpeer.log
MGG_AGG_PAIR=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:agg_gpair --launch-skip 8 -c 1 -o $O/pair_hostpeer_full python tools/hiding_b200.py --child --forms 1 --far 0.002 --reps 2 > $O/pair_hostpeer_full.log 2>&1
tail -2 $O/pair_hostpeer_full.log
MGG_BENCH_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --secondary none > $O/bench_2rank_1dev.json 2> $O/bench_2rank_1dev.err
tail -c 600 $O/bench_2rank_1dev.json; tail -3 $O/bench_2rank_1dev.err
