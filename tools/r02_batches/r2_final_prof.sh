# round-2 evidence refresh: launch list of the default bench command, ncu --set full of
# the dominant kernels (layer-1 K1, layer-2 K1 with ReLU on load, K2 X.W1, head)
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2fp; mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --secondary none > $O/launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"agg_group_hint|gemm_tc" --launch-skip 4 -c 4 -o $O/products_step python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --secondary none > $O/full.log 2>&1
tail -2 $O/full.log
