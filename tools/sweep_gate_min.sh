for v in 14 16 18 20; do for c in cfg5bt cfg2 cfg2bt cfg4bt cfg3bt cfg5cs; do
QCG_GATE_MIN_BITS=$v timeout 300 python bench.py --config $c --no-cpu --steps 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($v, '$c', round(d['ms_per_step'],4), d['gpu_launches'])"; done; done
