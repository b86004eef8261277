for F in "" "-DRD_MATCH_DEPTH=8" "-DRD_MATCH_DEPTH=12" "-DRD_MATCH_TILE=2" "-DRD_MATCH_DEPTH=8 -DRD_MATCH_TILE=2" ""; do
  RADE_EXTRA_NVCC_FLAGS="$F" python -m paper_2406_01467_b200.build --force > /dev/null 2>&1
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "
import json,sys
d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); k=d['config']['ms_per_view_by_kernel']
print('[$F]', round(d['value'],1), 'depth', round(k['depth_sort'],4), 'dup', round(k['duplicate'],4), 'tile', round(k['tile_sort'],4))"
done
