#!/bin/bash
# Decode attention at CaS-tail batch sizes (d=1 steps, 8 layers; event-bracketed per-class time)
for pt in "16 1024" "16 4096" "4 4096" "1 4096" "64 1024"; do
  set -- $pt
  env $EXTRA timeout 200 python bench.py --batch $1 --ctx $2 --layers 8 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --emulate-world 0 --cas-emulate 0 $WL 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.readline()); k=d['kernel_us_per_layer']; B=$1; S=$2
by=B*(S+1)*2*8*128*2*($WLAYERS)
print('B=$1 S_ctx=$2 $EXTRA attention us', k.get('attention'), 'GB/s', round(by/ (k.get('attention',1)*1e-6)/1e9))"
done
