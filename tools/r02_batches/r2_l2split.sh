cd $GRAFT_REPO_ROOT
O=gpurun_out/r2l2s; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o $O/l2_split_probe tools/l2_split_probe.cu || exit 1
for mb in 32 64 96 160; do timeout 120 $O/l2_split_probe $mb; done | tee $O/split.jsonl
for mode in 0 1 2; do
  timeout 300 ncu --metrics lts__t_sector_hit_rate.pct,dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:gather --launch-skip 1 -c 1 --csv $O/l2_split_probe 160 $mode 2>/dev/null | grep '^"' | sed "s/^/$mode,/" >> $O/ncu160.csv
done
cut -d, -f1,15- $O/ncu160.csv
