# round-2 final validation: GPU suite, smoke, bench (both arms)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2final; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -6 > $O/gputest.txt; cat $O/gputest.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; cat $O/smoke.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; python -c "import json;r=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);print(r['ms_per_step'], r['value'], r['roofline']['frac'], r['e2e']['value'], r['gpu_launches'], r['clocks'], r['secondary'][0]['ms_per_step'])"
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err; tail -c 300 $O/bench_ref.json
