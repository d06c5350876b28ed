cd $GRAFT_REPO_ROOT
O=gpurun_out/r2ef; mkdir -p $O
for ef in 0 1; do
  for gw in products-gcn reddit-gcn; do MGG_AGG_REMOTE_EF=$ef timeout 300 python tools/hiding_b200.py --graph $gw --device-peer --forms 1 --reps 3 --out $O/dev_${gw}_ef$ef.jsonl > /dev/null 2>&1; done
  MGG_AGG_REMOTE_EF=$ef timeout 400 python tools/hiding_b200.py --forms 1 --far 0.0005,0.002,0.01 --out $O/loc_ef$ef.jsonl > /dev/null 2>&1
  MGG_AGG_REMOTE_EF=$ef timeout 400 python tools/project_multi_gpu.py --workload products-gcn --parts 2,4,8 > $O/proj_ef$ef.jsonl 2>/dev/null
done
MGG_AGG_REMOTE_EF=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "pair_kernel or remote_fetch or phase" 2>&1 | tail -1
