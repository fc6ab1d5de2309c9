export SIDP_CAS_TIMEOUT_MS=5000
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "hybrid or serve_only or windowed" 2>&1 | tail -2
timeout 240 python bench.py --emulate-only --workload M3 --alias-owners --emulate-batch 1024 --emulate-ctx 384 --emulate-ce-share 0.3 --emulate-fetch-sms 12 --emulate-steps 2 > gpurun_out/hy_m3.log 2>&1; echo "m3 rc=$?"; grep -o '"ms_per_step": [0-9.]*\|"frac_T2": [0-9.]*\|"GBps": [0-9.]*\|Error.*' gpurun_out/hy_m3.log | head -5
