#!/bin/bash
# M3 (BASELINE configs[2]): Llama-3.1-70B WaS d=8 at the B_e region, max KV per GPU, owners
# aliased (bench --alias-owners) so the KV cache fits one GPU.  usage: bash tools/m3_be.sh "<pts>" "<variants>"
PTS=${1:-"1536:256 1024:384"}
VARS=${2:-"--slots=1,--slot-parts=2"}
for v in $VARS; do
  vv=${v//,/ }
  for pt in $PTS; do
    B=${pt%%:*}; C=${pt##*:}
    timeout 400 python bench.py --emulate-only --workload M3 --alias-owners --emulate-batch $B --emulate-ctx $C $vv 2>&1 | grep "^{\|Error" | python -c "
import json,sys
for ln in sys.stdin:
    if not ln.startswith('{'): print(ln.strip()[:300]); continue
    d=json.loads(ln); w=d['was_emulation']
    print('M3 B=$B ctx=$C $vv', round(w['ms_per_step'],2), 'ms T2', round(w['north_star_roofline']['frac_T2'],3), 'T3', round(w['north_star_roofline']['frac_T3'],3), 'fetch', round(w['fetch']['GBps'] or 0), 'tok/s rank', round(w['tokens_s_rank']), 'group', round(w['group_tokens_s_est']), w['kernel_us_per_layer'], 'slots GB', round(w['footprint_bytes_rank0']['slots']/1e9, 2))"
  done
done
