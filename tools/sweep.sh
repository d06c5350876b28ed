#!/bin/bash
# usage: tools/sweep.sh "ENV=..;ENV2=.." "ps dist wpb" ...   (runs on the GPU box)
envs="$1"; shift
for c in "$@"; do set -- $c
  for e in $(echo "$envs" | tr ';' ' '); do
    env $e python bench.py --steps 20 --warmup 5 --no-cpu --no-e2e --ps $1 --dist $2 --wpb $3 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$e', d['config']['ps'],d['config']['dist'],d['config']['wpb'], d['ms_per_step'], [o['ms'] for o in d['ops'] if o['kind'] in ('aggregate','dense')], d['clocks'].get('sm_mhz'), d['clocks'].get('reasons'))"
  done
done
