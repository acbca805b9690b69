python -c "from paper_1011_3077_b200 import build as b; b.build(force=True)"
for n in 512 1024; do for w in 0 1 2; do SDC_PANEL_WC=$w python tools/panel_bench.py $n > gpurun_out/pb6_w${w}_$n.txt 2>&1; done; done
SDC_PANEL_WC=2 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "panel or qr or config2 or config1" > gpurun_out/t9.log 2>&1; echo rc=$? >> gpurun_out/t9.log
