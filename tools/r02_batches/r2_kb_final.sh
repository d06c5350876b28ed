cd $GRAFT_REPO_ROOT
O=gpurun_out/r2kbf; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -1
timeout 600 python tools/hiding_b200.py --probe --forms 1,0 --far 0.0005,0.001,0.002,0.004,0.01,0.05 --out $O/hiding_locality.jsonl > /dev/null 2>&1
timeout 400 python tools/hiding_b200.py --forms 1 --far 0.001,0.004,0.01 --dim 64 --out $O/hiding_locality_d64.jsonl > /dev/null 2>&1
for n in 4 8; do timeout 400 python tools/hiding_b200.py --parts $n --forms 1 --far 0.0005,0.002,0.01 --out $O/fine_parts$n.jsonl > /dev/null 2>&1; done
for gw in config1 products-gcn reddit-gcn; do timeout 300 python tools/hiding_b200.py --graph $gw --device-peer --forms 1 --reps 3 --out $O/dev_$gw.jsonl > /dev/null 2>&1; done
timeout 600 python bench.py --no-cpu > $O/bench.json 2>/dev/null; python -c "import json;r=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);print(r['ms_per_step'], r['hiding']['hidden_remote_fraction'], r['hiding']['pipelined_vs_max_leg'])"
