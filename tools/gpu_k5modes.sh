#!/bin/bash
# bench lines for the K5 scheduling modes (C3, default otherwise): bash tools/gpu_k5modes.sh
for M in ${MODES:-set split batched set split}; do
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --k5 $M 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print('$M', round(d['value'],1), round(d['ms_per_step'],3))"
done
