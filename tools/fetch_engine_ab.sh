# WaS d=8 emulation: SM fetch kernel (48 CTAs, paced) vs copy engine (16 MB chunks, paced) at
# the B_e-regime batches where the layer compute shares the GPU with the fetch.
mkdir -p gpurun_out
for eng in sm ce; do
  for wl in "M2 1024 384" "M3 1024 64"; do
    set -- $wl
    timeout 600 python bench.py --workload $1 --emulate-only --emulate-batch $2 --emulate-ctx $3 --emulate-steps 3 --fetch $eng 2>&1 | tail -1 | \
      python -c "import json,sys; e=json.loads(sys.stdin.read())['was_emulation']; print('$eng', '$1', e['batch'], round(e['ms_per_step'],2), 'ms, fetch', round(e['fetch']['GBps'] or 0), 'GB/s busy', round(e['fetch']['fetch_busy_frac'] or 0, 3), 'T2 frac', round(e['north_star_roofline']['frac_T2'],3))" | tee -a gpurun_out/fetch_engine_ab.txt
  done
done
