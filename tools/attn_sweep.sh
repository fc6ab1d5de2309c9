# attention variants on the M2 shape: stages x CTA count (16 layers), then the full 64 layers
run() { env "$@" timeout 300 python bench.py --steps 5 --warmup 3 $LAYERS --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); r=d['roofline']; print('$* $LAYERS', 'ms/step', round(d['ms_per_step'],3), 'attn us', round(r['avg_launch_ms']*1e3,1), 'frac', round(r['frac'],3))"; }
LAYERS="--layers 16" run SIDP_ATTN_STAGES=2
LAYERS="--layers 16" run SIDP_ATTN_STAGES=3
LAYERS="" run SIDP_ATTN_STAGES=2
