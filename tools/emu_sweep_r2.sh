# Final r2 WaS d=8 emulation sweep: Qwen3-32B over the batch (largest context beside the 64
# emulated owner layers), whole vs tile-granular double-buffered slots, and the M3 points.
mkdir -p gpurun_out
for parts in 1 2; do
for bc in "256 1024" "512 768" "1024 384" "1536 256"; do
  set -- $bc
  timeout 600 python bench.py --emulate-only --cas-emulate 0 --m3-emulate 0 --emulate-steps 3 \
     --emulate-batch $1 --emulate-ctx $2 --slots 2 --slot-parts $parts 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); e=d['was_emulation']
if 'error' in e: print('B=$1', e); sys.exit()
print(json.dumps({'model': 'qwen3-32b', 'slot_parts': $parts, 'B': e['batch'], 'ctx': e['ctx'], 'ms': round(e['ms_per_step'],2),
  'group_est': round(e['group_tokens_s_est']), 'fetch_GBps': round(e['fetch']['GBps'] or 0),
  'frac_T2': round(e['north_star_roofline']['frac_T2'],3), 'frac_T3': round(e['north_star_roofline']['frac_T3'],3),
  'per_layer_median': round((e.get('per_remote_layer') or {}).get('frac_median', 0), 3)}))
" | tee -a gpurun_out/emu_sweep_r2.jsonl
done; done
bash tools/m3_be.sh "1024:384 1536:256" "--slots=2,--slot-parts=2 --slots=2" 2>&1 | sed "s/{'gate_up.*slots GB/slots GB/" | tee -a gpurun_out/emu_sweep_r2.jsonl
