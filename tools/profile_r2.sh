#!/bin/bash
# Round-2 evidence on one GPU box (gpurun): launch list of the M2 bench step, ncu --set full of
# the WaS fetch kernel as the ring runs it (alone: its SMs, DRAM bytes, duration), of attention
# and the GEMMs, and the NVLink metric names this ncu exposes (for the multi-GPU recipe).
mkdir -p gpurun_out
B="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --emulate-world 0 --cas-emulate 0"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 6000 --csv \
   --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1
echo "launches rc=$?"
timeout 600 env ONLY_RING=24 ncu --set full --clock-control none --import-source on -k regex:fetch_bulk -s 2 -c 1 \
   -o gpurun_out/prof_fetch -f python tools/fetch_bench.py > gpurun_out/ncu_fetch.log 2>&1
echo "fetch rc=$?"
python tools/fetch_bench.py > gpurun_out/fetch_bench.json 2>&1
S="python bench.py --steps 1 --warmup 3 --layers 4 --no-e2e --no-cpu-baseline --emulate-world 0 --cas-emulate 0"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"attn_(warp_)?kernel|gemm2_kernel|mlp2_kernel" -s 30 -c 5 \
   -o gpurun_out/prof_layer -f $S > gpurun_out/ncu_layer.log 2>&1
echo "layer rc=$?"
ncu --query-metrics 2>/dev/null | grep -i -E "nvl|nvlink|c2c" > gpurun_out/nvlink_metrics.txt
ncu --query-metrics-mode suffix --metrics nvlrx__bytes,nvltx__bytes 2>&1 | head -40 >> gpurun_out/nvlink_metrics.txt
nvidia-smi topo -m > gpurun_out/topo.txt 2>&1
ls -la gpurun_out
