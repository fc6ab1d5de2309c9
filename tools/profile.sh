#!/bin/bash
# Run on the GPU box (gpurun): launch list of the bench command + ncu --set full captures of the
# top kernels.  Outputs under gpurun_out/.
set -x
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --emulate-world 0"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv \
   --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
S="python bench.py --steps 1 --warmup 3 --layers 4 --no-e2e --no-cpu-baseline --emulate-world 0"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_(warp_)?kernel" -s 8 -c 1 \
   -o gpurun_out/prof_attn -f $S > gpurun_out/ncu_attn.log 2>&1
# one decoder layer's GEMMs (qkv, o, gate/up, down) after the warm-up layers, then the LM head
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gemm2_kernel|mlp2_kernel" -s 24 -c 4 \
   -o gpurun_out/prof_gemm -f $S > gpurun_out/ncu_gemm.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:"qkv_post|rmsnorm|resid_norm" -s 24 -c 4 \
   -o gpurun_out/prof_small -f $S > gpurun_out/ncu_small.log 2>&1
# the WaS fetch kernel inside the d=8 single-GPU emulation (2 launches)
E="python bench.py --steps 1 --warmup 3 --layers 16 --no-e2e --no-cpu-baseline --cas-emulate 0 --emulate-steps 1"
timeout 600 ncu --set full --clock-control none -k regex:fetch_kernel -s 20 -c 2 \
   -o gpurun_out/prof_fetch -f $E > gpurun_out/ncu_fetch.log 2>&1
ls -la gpurun_out
# ---- multi-GPU (skipped on a 1-GPU box): P2P fetch bandwidth of the ring's fetch kernel vs the
# LDG kernel and the copy engine, then the NVLink counters of one 24-SM fetch launch
if [ "$(python -c 'import torch; print(torch.cuda.device_count())')" -ge 2 ]; then
  python tools/nvlink_fetch_probe.py > gpurun_out/nvlink_fetch_probe.json 2>&1
  timeout 600 ncu --metrics gpu__time_duration.sum,nvlrx__bytes.sum,nvltx__bytes.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum \
     --clock-control none -k regex:fetch_bulk -s 2 -c 1 --csv --log-file gpurun_out/ncu_nvlink_fetch.csv \
     python tools/nvlink_fetch_probe.py --ctas 24 --reps 1 > gpurun_out/ncu_nvlink_fetch.log 2>&1
  # the d=N bench with NCCL's transport log (the control plane only: no collective on the data path)
  NCCL_DEBUG=INFO timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
     --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --steps 5 --warmup 3 \
     > gpurun_out/bench_2gpu.log 2>&1
fi
