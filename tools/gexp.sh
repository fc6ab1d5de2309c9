mkdir -p gpurun_out
export NO_CUBLAS=
python tools/gemm_bench.py 256 all 0 > gpurun_out/g_base.log 2>&1
NO_CUBLAS=1 SIDP_GEMM_KPS=1 python tools/gemm_bench.py 256 qkv,o,gate_up,down 0 > gpurun_out/g_kps1.log 2>&1
NO_CUBLAS=1 SIDP_GEMM_BNT=128 python tools/gemm_bench.py 256 qkv,o,gate_up,down 0 > gpurun_out/g_bnt128.log 2>&1
NO_CUBLAS=1 SIDP_GEMM_SW=2 python tools/gemm_bench.py 256 o,gate_up,down 0 > gpurun_out/g_sw2.log 2>&1
NO_CUBLAS=1 SIDP_GEMM_TRACE=1 python tools/gemm_bench.py 256 gate_up,down,o 0 > gpurun_out/g_trace.log 2>&1
tail -n 40 gpurun_out/g_*.log
