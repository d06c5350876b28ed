#!/bin/bash
# DRAM bytes per K1 launch of every fetch variant (ncu, one launch each).
OUT=${1:-gpurun_out/k1_fetch_ncu.csv}
: > "$OUT"
for wl in products-gcn orkut-gcn; do
  for v in "0 8" "64 8" "0 16" "64 16"; do
    set -- $v
    MGG_AGG_L2FETCH=$1 MGG_AGG_HINT_UNR=$2 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct \
      --clock-control none -k regex:agg_ --csv python tools/k1_fetch_sweep.py --child $wl --once 2>/dev/null \
      | grep '^"' | sed "s/^/$wl,$1,$2,/" >> "$OUT"
  done
done
cat "$OUT" | cut -c 1-250
