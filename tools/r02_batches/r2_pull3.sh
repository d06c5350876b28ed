cd $GRAFT_REPO_ROOT
O=gpurun_out/r2p3; mkdir -p $O
for m in ${MODES:-2 4}; do
  MGG_HALO_PULL_MODE=$m timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "halo_pull or shard_memory" 2>&1 | tail -1
  MGG_HALO_PULL_MODE=$m timeout 500 python tools/hiding_b200.py --fetch halo --forms 1 --far 0.0005,0.002,0.01,0.05 --out $O/loc_mode$m.jsonl > /dev/null 2>&1
  MGG_HALO_PULL_MODE=$m timeout 500 python tools/hiding_b200.py --fetch halo --parts 8 --forms 1 --far 0.0005,0.002,0.01 --out $O/loc8_mode$m.jsonl > /dev/null 2>&1
  MGG_HALO_PULL_MODE=$m MGG_HALO_FUSE=1 timeout 400 python tools/project_multi_gpu.py --workload products-gcn --parts 2,8 > $O/proj_mode$m.jsonl 2>/dev/null
done
