# round-2 batch 7: ReLU-on-load for HBM-resident hidden tables — GPU suite + bench
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2b7; mkdir -p $O
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -8 > $O/gputest.txt; cat $O/gputest.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; tail -c 2500 $O/bench.json | head -c 1400; echo
for wl in orkut-gcn products-gin; do timeout 600 python bench.py --workload $wl --secondary none --no-cpu > $O/bench_$wl.json 2> $O/bench_$wl.err; python -c "import json;r=json.loads(open('$O/bench_$wl.json').read().strip().splitlines()[-1]);print('$wl', r['ms_per_step'], r['value'], r['e2e']['value'], [(o['kind'],o['ms']) for o in r['ops']])"; done
