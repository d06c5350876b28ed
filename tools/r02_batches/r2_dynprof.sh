# ncu --set full of the pair kernel's local leg (phase 3), static vs dynamic schedule
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2dp; mkdir -p $O
for d in 0 1; do
  MGG_AGG_DYN=$d MGG_AGG_PAIR=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:agg_gpair --launch-skip 1 -c 1 -o $O/gpair_phase3_dyn$d python tools/hiding_b200.py --child --graph products-gcn --device-peer --forms 1 --reps 2 > $O/log_dyn$d.txt 2>&1
  tail -1 $O/log_dyn$d.txt
done
