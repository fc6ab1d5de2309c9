# Functional sweep of less-used bench configurations on one GPU (each must print a JSON line).
mkdir -p gpurun_out
run() { timeout 600 python bench.py "$@" 2>&1 | tail -1 | python -c "
import json,sys
try:
    d=json.loads(sys.stdin.read()); e=d.get('was_emulation',{})
    print('OK', ' '.join(sys.argv[1:]), d.get('ms_per_step'), e.get('ms_per_step'), e.get('error'))
except Exception as ex: print('FAIL', ' '.join(sys.argv[1:]), ex)" "$@"; }
run --workload M4 --emulate-only --emulate-batch 256 --emulate-ctx 256 --emulate-steps 2
run --workload M2 --emulate-only --pool ffn --emulate-batch 256 --emulate-ctx 512 --emulate-steps 2
run --workload M2 --emulate-only --order paper --slots 7 --emulate-batch 128 --emulate-ctx 512 --emulate-steps 2
run --workload M2 --emulate-only --emulate-world 4 --emulate-batch 256 --emulate-ctx 512 --emulate-steps 2
run --workload M2 --emulate-only --emulate-world 2 --slots 3 --emulate-batch 256 --emulate-ctx 512 --emulate-steps 2
run --workload M2 --steps 3 --warmup 3 --batch 64 --ctx 4096 --no-cpu-baseline --emulate-world 0 --cas-emulate 0
run --workload M2 --steps 3 --warmup 3 --batch 1 --ctx 2048 --no-cpu-baseline --emulate-world 0 --cas-emulate 0
