#!/bin/bash
# Emulation fidelity A/B: owner reads from local HBM (default) vs from a 32 MB L2 window
# (--l2-source: this GPU's HBM then carries only a real reader's traffic).
for v in "" "--l2-source"; do
  for pt in "M2 256 1024" "M2 1024 384" "M3 1024 384" "M3 1536 256"; do
    set -- $pt
    extra=""; [ "$1" = M3 ] && extra="--alias-owners"
    timeout 400 python bench.py --emulate-only --workload $1 --emulate-batch $2 --emulate-ctx $3 $extra $v 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); w=d['was_emulation']
print('$1 B=$2 ctx=$3 $v', round(w['ms_per_step'],2), 'ms T2', round(w['north_star_roofline']['frac_T2'],3), 'T3', round(w['north_star_roofline']['frac_T3'],3), 'fetch', round(w['fetch']['GBps'] or 0), 'group', round(w['group_tokens_s_est']), w['kernel_us_per_layer'])"
  done
done
