#!/bin/bash
# Round-1 refresh on one B200 (run under gpurun): GPU tests, every bench config, the ncu
# launch list of the config-5 twin (n=4096) and ncu --set full of the top kernels.
set -x
mkdir -p gpurun_out/refresh
python -c "from paper_1011_3077_b200 import build as b; b.build(force=True)"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/refresh/gpu_tests.log 2>&1; echo rc=$? >> gpurun_out/refresh/gpu_tests.log
timeout 900 python bench.py > gpurun_out/refresh/bench_default.json 2> gpurun_out/refresh/bench_default.err
for c in 1 2; do timeout 400 python bench.py --config $c --steps 5 --warmup 3 > gpurun_out/refresh/bench_c$c.json 2> gpurun_out/refresh/bench_c$c.err; done
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 > gpurun_out/refresh/bench_c3.json 2> gpurun_out/refresh/bench_c3.err
for c in 4 6 9; do timeout 900 python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/refresh/bench_c$c.json 2> gpurun_out/refresh/bench_c$c.err; done
for c in 7 8 10; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 > gpurun_out/refresh/bench_c$c.json 2> gpurun_out/refresh/bench_c$c.err; done
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/refresh/bench_reference.json 2> gpurun_out/refresh/bench_reference.err
L="python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline --config 5 --n 4096"
$L > gpurun_out/refresh/ncu_plain_launch.log 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/refresh/launches_cfg5_n4096.csv $L > gpurun_out/refresh/ncu_launch.log 2>&1
timeout 1200 bash tools/ncu_capture.sh > gpurun_out/refresh/ncu_capture.log 2>&1
