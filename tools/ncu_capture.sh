#!/bin/bash
# ncu --set full captures of the top kernels (run under gpurun; one GPU).
# Each profiled command is first run plain and must exit 0.
set -x
B="python tools/gemm_bench.py 8192"
$B > gpurun_out/ncu_plain_gemm.log 2>&1 || exit 1
# launch order of gemm_tn_tma_kernel in gemm_bench: square x7 first
ncu --set full --clock-control none --import-source on -k regex:gemm_tn_tma_kernel -s 2 -c 1 \
    -o gpurun_out/refresh/r01_gemm_square $B > gpurun_out/ncu_gemm_sq.log 2>&1
# rank-nb updates run in gemm_tn_tma_persist_kernel: launches rank-64 x7, rank-128 x7, rank-256 x7
ncu --set full --clock-control none --import-source on -k regex:gemm_tn_tma_persist -s 16 -c 1 \
    -o gpurun_out/refresh/r01_gemm_rank256 $B > gpurun_out/ncu_gemm_r256.log 2>&1
P="python tools/panel_bench.py 8192"
$P > gpurun_out/ncu_plain_panel.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:panel_qr -s 150 -c 1 \
    -o gpurun_out/refresh/r01_panel_grid $P > gpurun_out/ncu_panel_grid.log 2>&1
P2="python tools/panel_bench.py 1024"
$P2 > gpurun_out/ncu_plain_panel2.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:panel_qr -s 20 -c 1 \
    -o gpurun_out/refresh/r01_panel_cluster $P2 > gpurun_out/ncu_panel_cluster.log 2>&1
for f in gpurun_out/ncu_gemm_sq.log gpurun_out/ncu_gemm_r256.log gpurun_out/ncu_panel_grid.log gpurun_out/ncu_panel_cluster.log; do tail -n 2 $f; done
