#!/bin/bash
# Round bench refresh on the GPU box: every config's bench line + reference arms.
#   tools/refresh_bench.sh <tag>   -> gpurun_out/<tag>_bench_<cfg>.json, <tag>_ref_<cfg>.json
tag=${1:-r01}
mkdir -p gpurun_out
for c in cfg5bt cfg2 cfg1 cfg2bt cfg3bt cfg4bt cfg5cs cfg3cs cfg4 cfg2os cfg4os cfg5os cfg5; do
  timeout 900 python bench.py --config $c > gpurun_out/${tag}_bench_$c.json 2> gpurun_out/${tag}_bench_$c.err
done
for c in cfg5bt cfg1 cfg2 cfg2bt cfg4bt; do
  timeout 600 python bench.py --impl reference --config $c --steps 3 --warmup 1 > gpurun_out/${tag}_ref_$c.json 2>&1
done
