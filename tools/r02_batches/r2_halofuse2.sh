cd $GRAFT_REPO_ROOT
O=gpurun_out/r2hf2; mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "halo_pull or remote_fetch" 2>&1 | tail -1
for f in 1 0; do
  MGG_HALO_FUSE=$f timeout 600 python tools/hiding_b200.py --fetch halo --forms 1 --far 0.0005,0.002,0.01,0.05 --out $O/loc_halo_fuse$f.jsonl > /dev/null 2>&1
  for w in products-gcn orkut-gcn; do MGG_HALO_FUSE=$f timeout 400 python tools/project_multi_gpu.py --workload $w --parts 2,4,8; done > $O/projection_fuse$f.jsonl 2>/dev/null
done
