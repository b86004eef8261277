#!/bin/bash
# bench lines for alternative bench.py flag sets (C3): bash tools/gpu_flagsab.sh "<flags A>" "<flags B>" ...
for F in "$@"; do
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e $F 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print('[$F]', round(d['value'],1), round(d['ms_per_step'],3))"
done
