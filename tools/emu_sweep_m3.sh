# Llama-3.1-70B (M3) WaS d=8 single-GPU emulation over the batch: all 80 owner layers (137 GB)
# sit on this GPU, so only short contexts fit beside them.
mkdir -p gpurun_out
for bc in "256 256" "512 128" "1024 64" "1536 32"; do
  set -- $bc
  timeout 600 python bench.py --workload M3 --emulate-only --emulate-batch $1 --emulate-ctx $2 --emulate-steps 3 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); e=d['was_emulation']
print(json.dumps({'model': 'llama-3.1-70b', 'B': e['batch'], 'ctx': e['ctx'], 'ms': round(e['ms_per_step'],2), 'tok_s_rank': round(e['tokens_s_rank']),
  'group_est': round(e['group_tokens_s_est']), 'fetch_GBps': round(e['fetch']['GBps'] or 0), 'fetch_busy': round(e['fetch']['fetch_busy_frac'] or 0,3),
  'T2_ms': round(e['north_star_roofline']['T2_ms'],2), 'T3_ms': round(e['north_star_roofline']['T3_ms'],2),
  'frac_T2': round(e['north_star_roofline']['frac_T2'],3), 'frac_T3': round(e['north_star_roofline']['frac_T3'],3), 'us_layer': e['kernel_us_per_layer'],
  'kv_capacity_ratio': round(d['kv_capacity'].get('ratio', 0), 2)}))
" | tee -a gpurun_out/emu_sweep_m3.jsonl
done
