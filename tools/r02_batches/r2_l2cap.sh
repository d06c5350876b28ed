cd $GRAFT_REPO_ROOT
O=gpurun_out/r2l2; mkdir -p $O
timeout 600 python tools/l2_capacity_sweep.py > $O/sweep.jsonl 2> $O/sweep.err; cat $O/sweep.jsonl
for mb in 32 48 64 96 128 160; do
  timeout 300 ncu --metrics lts__t_sector_hit_rate.pct,dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum --clock-control none -k regex:gather_probe --launch-skip 1 -c 1 --csv python tools/l2_capacity_sweep.py --once $mb 2>/dev/null | grep '^"' | sed "s/^/$mb,/" >> $O/ncu.csv
done
cut -c1-40,180- $O/ncu.csv | head -40
