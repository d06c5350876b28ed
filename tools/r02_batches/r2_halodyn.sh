cd $GRAFT_REPO_ROOT
O=gpurun_out/r2hd; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multiprocess.py -m gpu -q -x -p no:cacheprovider -k "halo or shard_memory or multi or remote_fetch" 2>&1 | tail -1
for d in 1 0; do
  MGG_HALO_PULL_DYN=$d timeout 500 python tools/hiding_b200.py --fetch halo --forms 1 --far 0.0005,0.002,0.01,0.05 --out $O/loc_dyn$d.jsonl > /dev/null 2>&1
  MGG_HALO_PULL_DYN=$d timeout 500 python tools/hiding_b200.py --fetch halo --parts 8 --forms 1 --far 0.0005,0.002,0.01 --out $O/loc8_dyn$d.jsonl > /dev/null 2>&1
  MGG_HALO_PULL_DYN=$d MGG_HALO_FUSE=1 timeout 400 python tools/project_multi_gpu.py --workload products-gcn --parts 2,8 > $O/proj_fused_dyn$d.jsonl 2>/dev/null
done
timeout 300 python bench.py --no-cpu --no-e2e --secondary none --no-hiding > $O/bench.json 2>/dev/null; python -c "import json;r=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);print(r['ms_per_step'], r['roofline']['avg_launch_ms'])"
