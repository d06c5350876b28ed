# round-2 batch 3: GPU suite with the dynamic pair schedule default, hiding sweep
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2b3; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -8 > $O/gputest.txt; cat $O/gputest.txt
timeout 900 python tools/hiding_b200.py --probe --forms 1,2,0 --far 0.0005,0.001,0.002,0.004,0.01,0.05 --out $O/hiding_locality.jsonl > /dev/null 2>&1
timeout 600 python tools/hiding_b200.py --forms 1 --far 0.001,0.004,0.01 --dim 64 --out $O/hiding_locality_d64.jsonl > /dev/null 2>&1
timeout 1200 python tools/ablation_b200.py --slow-peer --out $O/ablation_slow_peer.jsonl > $O/ablation_slow_peer.log 2>&1
tail -c 400 $O/ablation_slow_peer.log
