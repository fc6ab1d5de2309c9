#!/bin/bash
one() { env $3 timeout 200 python bench.py --batch $1 --ctx $2 --layers 8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --emulate-world 0 --cas-emulate 0 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); k=d['kernel_us_per_layer']
by=$1*($2+1)*4096
print('B=$1 S_ctx=$2 $3 attention us', k.get('attention'), 'GB/s', round(by/(k.get('attention',1)*1e-6)/1e9))"; }
for c in 0 256 384; do one 16 1024 SIDP_ATTN_CTAS=$c; done
for c in 0 256 512; do one 16 4096 SIDP_ATTN_CTAS=$c; done
for c in 0 256; do one 32 1024 SIDP_ATTN_CTAS=$c; done
for c in 0 64 96; do one 1 1024 SIDP_ATTN_CTAS=$c; done
