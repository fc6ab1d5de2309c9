#!/bin/bash
# NEXT-3 A/B: WaS d=8 emulation with 2 whole-layer slots vs 1 tile-granular slot vs 1 whole-layer
# slot.  usage: bash tools/tile_ab.sh "256:1024 1024:384" [extra bench args]
PTS=${1:-"256:1024 1024:384"}
shift
for pt in $PTS; do
  B=${pt%%:*}; C=${pt##*:}
  for v in "--slots 2 --slot-parts 1" "--slots 1 --slot-parts 2" "--slots 1 --slot-parts 1" "--slots 2 --slot-parts 2"; do
    timeout 300 python bench.py --emulate-only --emulate-batch $B --emulate-ctx $C $v "$@" 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read()); w=d['was_emulation']
print('B=$B ctx=$C $v $*', round(w['ms_per_step'],2), 'ms T2', round(w['north_star_roofline']['frac_T2'],3), 'fetch', round(w['fetch']['GBps'] or 0), 'slot GB', round(w['footprint_bytes_rank0']['slots']/1e9,3), w['kernel_us_per_layer'])" || echo "B=$B $v failed"
  done
done
