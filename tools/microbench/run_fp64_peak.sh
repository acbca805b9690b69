#!/bin/bash
# FP64 peak microbenchmark with the SM clock sampled DURING the run (nvidia-smi every 100 ms):
# the DMMA / DFMA figures are only meaningful next to the clock they ran at.
set -e
cd "$(dirname "$0")"
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_peak fp64_peak.cu
smi=$(mktemp)
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv,noheader,nounits -lms 100 > "$smi" &
pid=$!
sleep 0.5
./fp64_peak ${1:-400000}
kill $pid; wait $pid 2>/dev/null || true
python3 - "$smi" <<'PY'
import statistics, sys
rows = [[c.strip() for c in l.split(",")] for l in open(sys.argv[1]) if l.strip()]
load = [r for r in rows if float(r[2]) > 200.0]          # samples under load (power > 200 W)
sm = [float(r[0]) for r in load] or [float(r[0]) for r in rows]
print(f"clocks during the run: sm_mhz median {statistics.median(sm):.0f} (min {min(sm):.0f}, max {max(sm):.0f}), "
      f"sm_max_mhz {rows[0][1]}, samples {len(rows)} ({len(load)} under load), "
      f"power max {max(float(r[2]) for r in rows):.0f} W, event reasons {sorted({r[3] for r in rows})}")
PY
