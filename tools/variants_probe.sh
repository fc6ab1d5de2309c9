export SIDP_CAS_TIMEOUT_MS=4000
run() { name=$1; shift; echo "== $name"; timeout 120 env "$@" python bench.py --workload M2 --emulate-only --layers 16 --emulate-batch 512 --emulate-ctx 768 --emulate-steps 2 > gpurun_out/var_$name.json 2> gpurun_out/var_$name.err; echo "rc=$?"; tail -c 300 gpurun_out/var_$name.err; python -c "
import json,sys
try:
  d=json.load(open('gpurun_out/var_$name.json'))['was_emulation']; print(d.get('ms_per_step'), d.get('fetch'), d.get('error'))
except Exception as e: print('no json', e)"; }
run base X=1
run nograph SIDP_GRAPH=0
run nowin SIDP_FETCH_WINDOW=0
run nograph_nowin SIDP_GRAPH=0 SIDP_FETCH_WINDOW=0
