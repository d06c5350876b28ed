# kind-split pair form (MGG_AGG_PAIR=4, agg_gsplit) vs agg_gpair (1)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2gs; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "pair_kernel_forms" 2>&1 | tail -3
timeout 900 python tools/hiding_b200.py --forms 1,4 --far 0.0005,0.002,0.01,0.05 --out $O/loc.jsonl > /dev/null 2>&1
timeout 600 python tools/hiding_b200.py --forms 1,4 --far 0.002,0.01 --dim 64 --out $O/loc_d64.jsonl > /dev/null 2>&1
for gw in config1 products-gcn reddit-gcn; do
  timeout 300 python tools/hiding_b200.py --graph $gw --device-peer --forms 1,4 --reps 3 --out $O/dev_${gw}.jsonl > /dev/null 2>&1
done
# sanitizer over the dynamic-schedule pair kernels
for pair in 1 4; do for tool in memcheck racecheck synccheck; do
  MGG_AGG_PAIR=$pair timeout 900 compute-sanitizer --tool $tool python tools/sanitize_pipe.py > $O/san_${pair}_$tool.txt 2>&1
  echo "pair=$pair $tool: $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|max row-relative' $O/san_${pair}_$tool.txt | tr '\n' ' ')"
done; done
