#!/bin/bash
# GEMM launch-knob sweep at one M (tools/gemm_bench.py, cold weights): default vs KPS=1 (twice the
# stages of half the size), token tile 128, and the k-block-major W layout.
M=${1:-256}; SH=${2:-qkv,o,down}
for v in "X=0" "SIDP_GEMM_KPS=1" "SIDP_GEMM_BNT=128" "SIDP_GEMM_KPS=1 SIDP_GEMM_BNT=128" "SIDP_GEMM_W_EVICT=0"; do
  env $v NO_CUBLAS=1 TAG="[$v]" python tools/gemm_bench.py $M $SH 0 2>&1 | grep -v Warn
done
python tools/gemm_bench.py $M $SH 0 2>&1 | grep cuBLAS
