cd $GRAFT_REPO_ROOT
O=gpurun_out/r2kb; mkdir -p $O
for lib in ${LIBS:-libmgg.so libmgg_kb8.so libmgg_kb128.so}; do
  MGG_LIB=$lib timeout 500 python tools/hiding_b200.py --forms 1 --far 0.0005,0.002,0.004,0.01 --out $O/loc_$lib.jsonl > /dev/null 2>&1
  MGG_LIB=$lib timeout 300 python tools/hiding_b200.py --graph products-gcn --device-peer --forms 1 --reps 3 --out $O/dev_$lib.jsonl > /dev/null 2>&1
done
