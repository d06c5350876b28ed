cd $GRAFT_REPO_ROOT
O=gpurun_out/r2ks; mkdir -p $O
for lib in libmgg.so libmgg_ks4.so libmgg_ks64.so; do
  MGG_LIB=$lib timeout 400 python tools/hiding_b200.py --forms 1 --far 0.0005,0.002,0.004 --out $O/loc_$lib.jsonl > /dev/null 2>&1
  MGG_LIB=$lib timeout 400 python tools/hiding_b200.py --parts 8 --forms 1 --far 0.0005,0.002 --out $O/loc8_$lib.jsonl > /dev/null 2>&1
  MGG_LIB=$lib timeout 300 python tools/hiding_b200.py --graph products-gcn --device-peer --forms 1 --reps 3 --out $O/dev_$lib.jsonl > /dev/null 2>&1
done
