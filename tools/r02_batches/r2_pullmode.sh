# halo pull modes: 1 interleaved per partition, 2 drained after each logical warp's partitions
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2pm; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "halo_pull or symmetric or shard_memory" 2>&1 | tail -1
MGG_HALO_PULL_MODE=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "halo_pull" 2>&1 | tail -1
for m in 1 2; do
  MGG_HALO_PULL_MODE=$m timeout 600 python tools/hiding_b200.py --fetch halo --forms 1 --far 0.0005,0.002,0.01,0.05 --out $O/loc_mode$m.jsonl > /dev/null 2>&1
  MGG_HALO_PULL_MODE=$m MGG_HALO_FUSE=1 timeout 400 python tools/project_multi_gpu.py --workload products-gcn --parts 2,8 > $O/proj_fused_mode$m.jsonl 2>/dev/null
done
