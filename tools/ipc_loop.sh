#!/bin/bash
# Repeats the two-process CUDA-IPC test N times per K1 pair-kernel setting and
# counts failures (50 consecutive clean runs).
# usage: tools/ipc_loop.sh N [out]
N=${1:-10}; OUT=${2:-gpurun_out/ipc_loop.txt}
mkdir -p "$(dirname "$OUT")"; : > "$OUT"
for pair in ${PAIRS:-1}; do
  fails=0
  for i in $(seq 1 "$N"); do
    if MGG_AGG_PAIR=$pair timeout 600 python -m pytest tests/test_gpu_multiprocess.py -x -q -m gpu \
        -p no:cacheprovider > /tmp/ipc_$pair_$i.log 2>&1; then :; else
      fails=$((fails+1)); echo "--- MGG_AGG_PAIR=$pair iter $i FAILED" >> "$OUT"; tail -30 /tmp/ipc_$pair_$i.log >> "$OUT"
    fi
  done
  echo "MGG_AGG_PAIR=$pair: $fails failures in $N runs (3 cases each)" >> "$OUT"
done
cat "$OUT"
