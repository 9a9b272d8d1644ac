#!/bin/bash
# GPU-box check: parity tests, then a short bench per config and (optionally) an ncu
# launch list per config. Usage (under gpurun):  bash tools/gpu_check.sh [launches]
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for c in c1 c2 c3 c4 c5; do
    timeout 300 python bench.py --workload $c --steps 20 --warmup 5 --no-cpu-baseline --stages \
        > gpurun_out/plain_$c.log 2> gpurun_out/stages_$c.log
    python - "$c" <<'EOF'
import json, sys
c = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/plain_{c}.log").read().strip().splitlines()[-1])
    print(c, "value ms %.4f" % d["ms_per_step"], "e2e ms %.4f" % d["e2e"]["value"],
          "launches", d["gpu_launches"], "roof", d.get("roofline", {}).get("frac"))
except Exception as e:
    print(c, "FAILED", e)
EOF
done
if [ "${1:-}" = "launches" ]; then
    for c in c1 c2 c3 c4 c5; do
        timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
            --log-file gpurun_out/launches_$c.csv python bench.py --workload $c --steps 3 --warmup 3 \
            --no-cpu-baseline > /dev/null 2>&1
        python tools/launch_summary.py gpurun_out/launches_$c.csv 2>/dev/null | head -14
    done
fi
