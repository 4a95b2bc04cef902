#!/bin/bash
# power / clock during DMMA-heavy (full DP) vs 3xTF32-heavy (MP t=2) factorizations
mkdir -p gpurun_out
for args in "--n 49152 --dp" "--n 98304 --t 2"; do
  nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.sw_power_cap --format=csv,noheader -lms 100 > /tmp/pw.csv &
  sp=$!
  timeout 300 python tools/kbench.py $args --lookahead 1 2>&1 | grep -E "cholesky|upd"
  kill $sp
  python - <<'PY'
import statistics
rows=[l.split(', ') for l in open('/tmp/pw.csv') if l.strip()]
rows=[r for r in rows if float(r[2].split()[0])>300]
ck=[float(r[1].split()[0]) for r in rows]; pw=[float(r[2].split()[0]) for r in rows]
print(f"   under load: {len(rows)} samples, sm clock median {statistics.median(ck):.0f} MHz (min {min(ck):.0f}), power median {statistics.median(pw):.0f} W (max {max(pw):.0f}), power-capped samples {sum('Active' in r[3] for r in rows)}")
PY
done
