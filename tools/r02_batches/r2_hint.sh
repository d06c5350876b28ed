# L2-hinted gpair (MGG_AGG_PAIR_HINT=1 default) vs plain
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2h; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "pair_kernel_forms or remote_fetch or phase or full_size" 2>&1 | tail -2
for h in 0 1; do
  MGG_AGG_PAIR_HINT=$h timeout 600 python tools/hiding_b200.py --forms 1 --far 0.0005,0.002,0.01 --out $O/loc_hint$h.jsonl > /dev/null 2>&1
  for gw in products-gcn reddit-gcn config1; do
    MGG_AGG_PAIR_HINT=$h timeout 300 python tools/hiding_b200.py --graph $gw --device-peer --forms 1 --reps 3 --out $O/dev_${gw}_hint$h.jsonl > /dev/null 2>&1
  done
done
