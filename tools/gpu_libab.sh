#!/bin/bash
# A/B of prebuilt libraries (RADE_LIB): bash tools/gpu_libab.sh <lib A> <lib B> ... (alternating runs)
for L in "$@"; do
  RADE_LIB=$L timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); k=d['config']['ms_per_view_by_kernel']
print('[$L]', round(d['value'],1), 'fwd', round(k['render_fwd'],4), 'bwd', round(k['render_bwd'],4), 'pre', round(k['preprocess_fwd'],4), 'prebwd', round(k['preprocess_bwd'],4))"
done
