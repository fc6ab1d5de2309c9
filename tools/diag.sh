export SIDP_CAS_TIMEOUT_MS=3000
timeout 120 python tools/ring_diag.py --layers 16 --steps 6 > gpurun_out/rd_graph.log 2>&1; echo "graph rc=$?"; tail -50 gpurun_out/rd_graph.log
SIDP_GRAPH=0 timeout 120 python tools/ring_diag.py --layers 16 --steps 6 > gpurun_out/rd_eager.log 2>&1; echo "eager rc=$?"; tail -12 gpurun_out/rd_eager.log
timeout 120 python tools/ring_diag.py --layers 16 --steps 6 --sync-each > gpurun_out/rd_graph_sync.log 2>&1; echo "graph_sync rc=$?"; tail -30 gpurun_out/rd_graph_sync.log
