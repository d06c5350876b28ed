cd $GRAFT_REPO_ROOT
O=gpurun_out/r2hf3; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multiprocess.py -m gpu -q -x -p no:cacheprovider -k "halo or remote_fetch or shard_memory or multi or cfg5 or full_size" 2>&1 | tail -1
timeout 600 python tools/hiding_b200.py --fetch halo --forms 1 --far 0.0005,0.001,0.002,0.004,0.01,0.05 --out $O/loc_halo_auto.jsonl > /dev/null 2>&1
timeout 600 python tools/hiding_b200.py --fetch halo --forms 1 --far 0.002,0.01 --dim 64 --out $O/loc_halo_auto_d64.jsonl > /dev/null 2>&1
for w in products-gcn orkut-gcn; do timeout 400 python tools/project_multi_gpu.py --workload $w --parts 2,8; done > $O/projection_auto.jsonl 2>/dev/null; cat $O/projection_auto.jsonl | cut -c1-200
