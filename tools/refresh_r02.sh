#!/bin/bash
# Round-2 refresh on one B200 (run under gpurun): smoke, GPU tests and every bench config.
# (ncu: tools/ncu_capture.sh and the launch list are separate runs.)
set -x
OUT=gpurun_out/${REFRESH_TAG:-refresh_r02}
mkdir -p $OUT
python -c "from paper_1011_3077_b200 import build as b; b.build(force=True)"
python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1
if [ -z "$SKIP_TESTS" ]; then
timeout 1500 python -m pytest tests -m gpu -q --durations=15 > $OUT/gpu_tests.log 2>&1; echo rc=$? >> $OUT/gpu_tests.log
fi
timeout 900 python bench.py > $OUT/bench_default.json 2> $OUT/bench_default.err
timeout 400 python bench.py --config 1 --steps 2000 --warmup 20 > $OUT/bench_c1.json 2> $OUT/bench_c1.err   # long enough for the clock sampler
for c in 2; do timeout 400 python bench.py --config $c --steps 5 --warmup 3 > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err; done
timeout 600 python bench.py --config 3 --steps 3 --warmup 3 > $OUT/bench_c3.json 2> $OUT/bench_c3.err
for c in 4 6 9; do timeout 900 python bench.py --config $c --steps 1 --warmup 3 --no-cpu-baseline > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err; done
for c in 7 8 10; do timeout 600 python bench.py --config $c --steps 3 --warmup 3 > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err; done
timeout 600 python bench.py --config 8 --leaf 1 --steps 2 --warmup 1 > $OUT/bench_c8_leaf1.json 2> $OUT/bench_c8_leaf1.err
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
tail -n 3 $OUT/gpu_tests.log; cat $OUT/bench_default.json
