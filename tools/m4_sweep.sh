# BASELINE configs[3] (M4) analogue: Qwen2.5-72B WaS at d = 2/4/8 (single-GPU emulation), cache
# slots 2-4, B = 256, S_ctx = 256 (the 80 owner layers, 140 GB, sit on this one GPU).
mkdir -p gpurun_out
for d in 2 4 8; do for s in 2 3 4; do
  timeout 600 python bench.py --workload M4 --emulate-only --emulate-world $d --slots $s --emulate-batch 256 --emulate-ctx 256 --emulate-steps 3 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); e=d['was_emulation']
print(json.dumps({'model': 'qwen2.5-72b', 'd': e['world_emulated'], 'slots': e['slots'], 'B': e['batch'], 'ctx': e['ctx'], 'ms': round(e['ms_per_step'],2),
  'group_est': round(e['group_tokens_s_est']), 'fetch_GBps': round(e['fetch']['GBps'] or 0), 'fetch_busy': round(e['fetch']['fetch_busy_frac'] or 0,3),
  'T2_ms': round(e['north_star_roofline']['T2_ms'],2), 'frac_T2': round(e['north_star_roofline']['frac_T2'],3), 'kv_ratio': round(d['kv_capacity'].get('ratio',0),2)}))
" | tee -a gpurun_out/m4_sweep.jsonl
done; done
