#!/bin/bash
# ncu --set full captures of the top kernels on a mid-size step (run under gpurun).
# Each command first runs plain (must exit 0), then under ncu.
set -x
CMD="python bench.py --config 5 --n 4096 --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
$CMD > gpurun_out/ncu_plain.log 2>&1 || exit 1
# square n x n GEMM (IRS a5), rank-256 update, split-K W0, panel kernel (grid and cluster)
ncu --set full --clock-control none --import-source on -k regex:gemm_tn_tma_kernel -s 40 -c 6 \
    -o gpurun_out/r01_gemm $CMD > gpurun_out/ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:panel_qr_kernel -s 10 -c 2 \
    -o gpurun_out/r01_panel $CMD > gpurun_out/ncu_panel.log 2>&1
tail -2 gpurun_out/ncu_gemm.log gpurun_out/ncu_panel.log
