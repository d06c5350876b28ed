# round-2 bench lines for every workload (product arm, device + e2e; CPU port skipped)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2all; mkdir -p $O
for w in config1 reddit-gcn products-gcn products-gin orkut-gcn reddit-gcn-norm reddit-rmat-gcn products-rmat-gin orkut-rmat-gcn; do
  timeout 600 python bench.py --workload $w --secondary none --no-cpu > $O/$w.json 2> $O/$w.err
  python -c "import json;r=json.loads(open('$O/$w.json').read().strip().splitlines()[-1]);print('$w', r['ms_per_step'], r['value'], r['e2e']['value'], r['roofline'].get('bound'), r['roofline'].get('frac'), r['roofline']['kernel'][:60])"
done
