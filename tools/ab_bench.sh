#!/bin/bash
# A/B of environment switches on the headline bench (no extras, no CPU leg):
#   tools/ab_bench.sh "NAME ENV=.. ENV=.." ...   -> one line per variant per repeat
variants=("$@")
for rep in 1 2; do
for v in "${variants[@]}"; do
  read -r name envs <<< "$v"
  line=$(env $envs timeout 600 python bench.py --no-cpu-baseline --no-extras --steps 20 2>/dev/null | tail -1)
  python -c "
import json,sys; d=json.loads(sys.argv[2]); print('%-14s %.4f ms  %.1f M pts/s  e2e %.1f M  sweeps %s' % (sys.argv[1], d['ms_per_step'], d['value']/1e6, d['e2e']['value']/1e6, d.get('psh_sweeps')))" "$name" "$line"
done; done
