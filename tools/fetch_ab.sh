#!/bin/bash
# A/B of the WaS fetch transport in the d=8 single-GPU emulation (bench.py --emulate-only):
# the SM bulk fetch (optionally under env variants) vs the copy engine, over batch / context.
# usage: bash tools/fetch_ab.sh "256:1024 512:768 1024:384" "base SIDP_BULK_CFG=24x8" [extra bench args]
PTS=${1:-"256:1024 512:768 1024:384"}
VARS=${2:-"base"}
shift 2
summ() { python -c "import json,sys
for ln in sys.stdin:
    if ln.startswith('{'):
        d=json.loads(ln); w=d['was_emulation']
        print('$1', round(w['ms_per_step'],2), 'ms T2', round(w['north_star_roofline']['frac_T2'],3), 'fetch', round(w['fetch']['GBps'] or 0), w['kernel_us_per_layer'])"; }
for pt in $PTS; do
  B=${pt%%:*}; C=${pt##*:}
  for v in $VARS; do
    if [ "$v" = base ]; then e=""; else e="$v"; fi
    env $e timeout 200 python bench.py --emulate-only --emulate-batch $B --emulate-ctx $C "$@" 2>&1 | summ "B=$B ctx=$C sm $v"
  done
  timeout 200 python bench.py --emulate-only --emulate-batch $B --emulate-ctx $C --fetch ce "$@" 2>&1 | summ "B=$B ctx=$C ce"
done
