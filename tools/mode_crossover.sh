# CaS vs WaS crossover (PAPER.md:232 B_th, SURVEY.md M5 analogue) on the Qwen3-32B shape, d=8
# emulated on one GPU, S_ctx = 256: CaS all-live per-rank batches vs the WaS emulation.
mkdir -p gpurun_out
CAS_BATCHES=16,32,64,128 CAS_CTX=256 timeout 900 python tools/cas_emu_check.py 64 8 2>&1 | tail -1 > gpurun_out/cas_cross.txt
for B in 16 64 128 256; do
  timeout 600 python bench.py --emulate-only --emulate-batch $B --emulate-ctx 256 --emulate-steps 3 2>&1 | tail -1 | \
    python -c "import json,sys; e=json.loads(sys.stdin.read())['was_emulation']; print('WaS B=%d ctx=%d %.2f ms' % (e['batch'], e['ctx'], e['ms_per_step']))" >> gpurun_out/cas_cross.txt
done
cat gpurun_out/cas_cross.txt
