mkdir -p gpurun_out
for cfg in "SIDP_GEMM_PARTIAL=0" "SIDP_GEMM_PART_SW_MIN_M=0"; do
env $cfg timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none -c 200 --csv --log-file gpurun_out/l_$(echo $cfg|tr '=' '_').csv python bench.py --steps 1 --warmup 3 --layers 4 --no-e2e --no-cpu-baseline > /dev/null 2>&1
done
ls gpurun_out
