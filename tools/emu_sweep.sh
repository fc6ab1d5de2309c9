# WaS d=8 single-GPU emulation over the batch (B_e analysis, SURVEY.md §8(d) M3 analogue on the
# Qwen3-32B shape): largest context that fits beside the 64 emulated owner layers.
mkdir -p gpurun_out
for bc in "256 1024" "512 768" "768 512" "1024 384" "1536 256"; do
  set -- $bc
  timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e \
     --emulate-batch $1 --emulate-ctx $2 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); e=d['was_emulation']
if 'error' in e: print('B=$1', e); sys.exit()
print(json.dumps({'B': e['batch'], 'ctx': e['ctx'], 'ms': round(e['ms_per_step'],2), 'tok_s_rank': round(e['tokens_s_rank']),
  'group_est': round(e['group_tokens_s_est']), 'fetch_GBps': round(e['fetch']['GBps'] or 0), 'fetch_busy': round(e['fetch']['fetch_busy_frac'] or 0,3),
  'T2_ms': round(e['north_star_roofline']['T2_ms'],2), 'T3_ms': round(e['north_star_roofline']['T3_ms'],2),
  'frac_T2': round(e['north_star_roofline']['frac_T2'],3), 'frac_T3': round(e['north_star_roofline']['frac_T3'],3), 'us_layer': e['kernel_us_per_layer']}))
" | tee -a gpurun_out/emu_sweep.jsonl
done
