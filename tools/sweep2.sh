#!/bin/bash
# usage: tools/sweep2.sh "ENV=..;ENV2=.." workload ...  (GPU box) — per-op ms for each env x workload
envs="$1"; shift
for w in "$@"; do
  for e in $(echo "$envs" | tr ';' ' '); do
    env $e python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$e', '$w', d['ms_per_step'], [(o['kind'][:3],o['width'],o['ms']) for o in d['ops'] if o['kind'] in ('aggregate','dense','dense_chain')])"
  done
done
