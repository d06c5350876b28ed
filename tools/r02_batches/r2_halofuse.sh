# fused halo pull: parity, slow-peer hiding, same-device per-part K1, bench regression check
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2hf; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "halo or remote_fetch or full_size or cfg5 or phase or shard_memory or multi_gpu" 2>&1 | tail -2
for f in 1 0; do
  MGG_HALO_FUSE=$f timeout 600 python tools/hiding_b200.py --fetch halo --forms 1 --far 0.0005,0.002,0.01,0.05 --out $O/loc_halo_fuse$f.jsonl > /dev/null 2>&1
  MGG_HALO_FUSE=$f timeout 300 python tools/hiding_b200.py --fetch halo --graph config1 --forms 1 --reps 3 --ps 8 --dist 8 --wpb 2 --out $O/config1_halo_hostpeer_fuse$f.jsonl > /dev/null 2>&1
  for w in products-gcn orkut-gcn reddit-gcn; do MGG_HALO_FUSE=$f timeout 400 python tools/project_multi_gpu.py --workload $w --parts 2,4,8; done > $O/projection_fuse$f.jsonl 2>/dev/null
done
timeout 600 python bench.py --secondary reddit-gcn --no-e2e --no-cpu > $O/bench.json 2> $O/bench.err; python -c "import json;r=json.loads(open('$O/bench.json').read().strip().splitlines()[-1]);print(r['ms_per_step'], r['roofline']['avg_launch_ms'], [(o['kind'],o['ms']) for o in r['ops']], r['secondary'][0]['ms_per_step'])"
timeout 900 tools/ipc_loop.sh 5 $O/ipc_loop.txt > /dev/null 2>&1; tail -1 $O/ipc_loop.txt
