#!/bin/bash
# ms/step of a list of bench configs (no CPU baseline), one line each:  tools/quick_bench.sh cfg5bt cfg2 ...
for c in "$@"; do
  timeout 300 python bench.py --config $c --no-cpu --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c', round(d['ms_per_step'],4), d['roofline']['kernel'], round(d['roofline']['frac'],3))"
done
