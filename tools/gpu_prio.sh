python -c "import torch; print('prio range', torch.cuda.Stream.priority_range())"
for P in none views views-k5 none views; do
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --prio $P 2>/dev/null | python -c "import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][0]); print('$P', round(d['value'],1), d['ms_per_step'])"
done
