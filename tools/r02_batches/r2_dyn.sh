# dynamic ticket schedule of agg_gpair (MGG_AGG_DYN) vs the static schedule
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2dyn; mkdir -p $O
for d in ${DYNS:-0 4 8 16 32}; do
  MGG_AGG_DYN=$d timeout 600 python tools/hiding_b200.py --forms 1 --far 0.0005,0.002,0.01,0.05 --out $O/loc_dyn$d.jsonl > /dev/null 2>&1
  for gw in config1 products-gcn reddit-gcn; do
    MGG_AGG_DYN=$d timeout 300 python tools/hiding_b200.py --graph $gw --device-peer --forms 1 --reps 3 --out $O/dev_${gw}_dyn$d.jsonl > /dev/null 2>&1
  done
done
MGG_AGG_DYN=1 timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "pair or fine or multi or phase or remote" 2>&1 | tail -3
