#!/bin/bash
# CaS ladder timing (bench.py --cas-only, 8 virtual ranks): V3 (default) vs V2 vs V1.
# usage: bash tools/cas_ab.sh "<variants>" [extra bench args]
VARS=${1:-"SIDP_CAS_FUSED=2 SIDP_CAS_FUSED=1 SIDP_CAS_FUSED=0"}
shift
for v in $VARS; do
  env $v timeout 400 python bench.py --cas-only "$@" 2>&1 | grep '^{' | python -c "
import json,sys
d=json.loads(sys.stdin.read())['cas_emulation']
print('$v', [(r['pattern'], round(r['ms_per_layer']*1e3,1), round(r['host_enqueue_ms'],1)) for r in d.get('results',[])], d.get('timeouts'), d.get('one_live_kernel_us_per_layer'), d.get('error',''))"
done
