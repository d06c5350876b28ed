cd $GRAFT_REPO_ROOT
for s in 228 132; do timeout 300 python tools/fuzz_repro.py $s 3 2>&1 | tail -1; done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "dense or gin or gcn or full_size or chain" 2>&1 | tail -2
for i in 1 2; do MGG_FUZZ_N=300 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k fuzz_forward --tb=short 2>&1 | grep -E "^E |passed|failed" | head -4; done
timeout 600 python bench.py --no-cpu --no-e2e > gpurun_out/k2acc_bench.json 2>/dev/null; python -c "import json;r=json.loads(open('gpurun_out/k2acc_bench.json').read().strip().splitlines()[-1]);print(r['ms_per_step'], [(o['kind'],o['ms']) for o in r['ops']], r['secondary'][0]['ms_per_step'])"
timeout 300 python bench.py --workload products-gin --no-cpu --no-e2e --secondary none > gpurun_out/k2acc_gin.json 2>/dev/null; python -c "import json;r=json.loads(open('gpurun_out/k2acc_gin.json').read().strip().splitlines()[-1]);print(r['ms_per_step'], [(o['kind'],o['ms']) for o in r['ops'] if o['kind']!='aggregate'])"
