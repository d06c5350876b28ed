# round-2 batch 2: remote-latency hiding (host-mapped slow peer), ablations
# (same-device and slow-peer), the two-process IPC loop
set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2b2; mkdir -p $O
timeout 1500 python tools/hiding_b200.py --probe --forms 1,2,3,0 --out $O/hiding_locality.jsonl > $O/hiding_locality.log 2>&1
tail -c 1500 $O/hiding_locality.log
for gw in config1 products-gcn reddit-gcn; do
  timeout 600 python tools/hiding_b200.py --graph $gw --device-peer --forms 1,2,3,0 --reps 3 --out $O/hiding_devpeer_$gw.jsonl > /dev/null 2>&1
done
timeout 300 python tools/hiding_b200.py --graph config1 --forms 1,2,3,0 --reps 3 --ps 8 --dist 8 --wpb 2 --out $O/hiding_hostpeer_config1.jsonl > /dev/null 2>&1
timeout 1200 python tools/ablation_b200.py --slow-peer --out $O/ablation_slow_peer.jsonl > $O/ablation_slow_peer.log 2>&1
tail -c 1500 $O/ablation_slow_peer.log
timeout 1500 python tools/ablation_b200.py --out $O/ablation.jsonl > $O/ablation.log 2>&1
tail -c 600 $O/ablation.log
timeout 1800 tools/ipc_loop.sh 30 $O/ipc_loop.txt > /dev/null 2>&1
tail -3 $O/ipc_loop.txt
