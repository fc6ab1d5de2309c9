#!/bin/bash
# Round-2 final evidence (gpurun, one GPU): the M2 bench step's launch list (durations + DRAM
# bytes per launch, cold and serialised) and ncu --set full of one decoder layer's kernels
# (attention, QKV / O GEMMs, fused MLP, qkv_post, the fix-ups) after the warm-up layers.
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --emulate-world 0 --cas-emulate 0 --m3-emulate 0"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv \
   --log-file gpurun_out/launches_r2b.csv $B > gpurun_out/ncu_launches_r2b.log 2>&1
echo "launches rc=$?"
S="python bench.py --steps 1 --warmup 3 --layers 4 --no-e2e --no-cpu-baseline --emulate-world 0 --cas-emulate 0 --m3-emulate 0"
timeout 900 ncu --set full --clock-control none --import-source on \
   -k regex:"attn_(warp_)?kernel|gemm2_kernel|mlp2_kernel|qkv_post|resid_norm" -s 42 -c 7 \
   -o gpurun_out/prof_layer_r2b -f $S > gpurun_out/ncu_layer_r2b.log 2>&1
echo "layer rc=$?"
