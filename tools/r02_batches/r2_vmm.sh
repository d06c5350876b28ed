# symmetric VMM stores: GPU suite, bench, fine-mode flat vs table addressing
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2vmm; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_parity.py -k "symmetric or pair_kernel or halo" -m gpu -q -p no:cacheprovider 2>&1 | tail -6 > $O/gputest.txt; cat $O/gputest.txt
timeout 600 python bench.py --no-cpu > $O/bench.json 2> $O/bench.err; python -c "import json;r=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);print(r['ms_per_step'], r['value'], r['roofline']['frac'], r['e2e']['value'], r['secondary'][0]['ms_per_step'])"
for v in "1 1" "0 1"; do set -- $v
  MGG_VMM=$1 MGG_FLAT=$2 timeout 300 python tools/hiding_b200.py --graph products-gcn --device-peer --forms 1 --reps 3 --out $O/dev_products_vmm$1_flat$2.jsonl > /dev/null 2>&1
  MGG_VMM=$1 MGG_FLAT=$2 timeout 300 python tools/project_multi_gpu.py --workload products-gcn --parts 2,8 > $O/proj_vmm$1_flat$2.jsonl 2>/dev/null
done
