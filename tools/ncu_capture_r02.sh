#!/bin/bash
# Round-2 ncu evidence (run under gpurun; one GPU).  Each profiled command is first run plain.
set -x
OUT=gpurun_out/ncu_r02
REP=/tmp/ncu_r02_reps   # .ncu-rep files stay on the box (gpurun_out is limited to 64 MiB): summaries only
mkdir -p $OUT $REP
python -c "from paper_1011_3077_b200 import build as b; b.build(force=True)"
# (1) launch list of the headline command, bounded to the first launches (ncu serialises every launch)
H="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline"
if [ -z "$SKIP_LIST" ]; then
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c ${NCU_COUNT:-16000} --csv --log-file $OUT/launches_default.csv $H > $OUT/ncu_list.log 2>&1
python tools/summarize_launches.py $OUT/launches_default.csv "ncu --metrics gpu__time_duration.sum --clock-control none -c ${NCU_COUNT:-16000} --csv: $H (headline workload: config 5, n=16384; first launches only)" > $OUT/launches_default.txt
gzip -f $OUT/launches_default.csv
fi
# (2) --set full of the top kernels
B="python tools/gemm_bench.py 8192"
$B > $OUT/plain_gemm.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:gemm_tn_tma_kernel -s 2 -c 1 -o $REP/r02_gemm_square $B > $OUT/ncu_sq.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:gemm_tn_tma_persist -s 16 -c 1 -o $REP/r02_gemm_rank256 $B > $OUT/ncu_r256.log 2>&1
P="python tools/panel_bench.py 8192"
SDC_CQ_SPLIT=2 $P > $OUT/plain_panel.log 2>&1 || exit 1
for k in k_cqs_gram k_cqs_mid1 k_cqs_q1 k_cqs_mid2 k_cqs_y; do
  SDC_CQ_SPLIT=2 ncu --set full --clock-control none --import-source on -k regex:$k -s 40 -c 1 -o $REP/r02_$k $P > $OUT/ncu_$k.log 2>&1
done
SDC_CQ_SPLIT=0 $P > $OUT/plain_panel_cluster.log 2>&1
SDC_CQ_SPLIT=0 ncu --set full --clock-control none --import-source on -k regex:panel_qr -s 40 -c 1 -o $REP/r02_panel_mcluster_cqr $P > $OUT/ncu_panel.log 2>&1
S="python bench.py --config 8 --leaf 1 --n 512 --steps 1 --warmup 0 --no-cpu-baseline"
$S > $OUT/plain_schur.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:k_schur_leaves -s 1 -c 1 -o $REP/r02_k_schur_leaves $S > $OUT/ncu_schur.log 2>&1
python tools/ncu_summary.py $REP/*.ncu-rep > $OUT/ncu_full_summary.txt 2>&1
rm -rf $REP
ls -la $OUT
