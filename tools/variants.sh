#!/bin/bash
# Compare engine build variants (build_var/<v>/libqcut_gpu.so) on the GPU box:
#   tools/variants.sh "a b c" [configs]
# Prints ms_per_step and the dominant launch per variant and config.
vars=${1:-a}
cfgs=${2:-cfg2}
mkdir -p gpurun_out
for v in $vars; do
  for c in $cfgs; do
    QCUT_GPU_LIB=build_var/$v/libqcut_gpu.so timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu \
      > gpurun_out/var_${v}_${c}.json 2> gpurun_out/var_${v}_${c}.err
    python - "$v" "$c" <<'PY'
import json, sys
v, c = sys.argv[1:3]
try:
    r = json.loads(open(f"gpurun_out/var_{v}_{c}.json").read().strip().splitlines()[-1])
    rf = r["roofline"]
    print(f"{v} {c} ms_per_step={r['ms_per_step']:.4f} s_amp={r.get('s_per_amplitude')} dom={rf.get('kernel')} "
          f"dom_ms={rf['dominant_ms']:.4f} frac={rf['frac']:.3f} amp={r.get('amplitude',{}).get('abs2')}")
except Exception as e:
    print(v, c, "FAILED", e, open(f"gpurun_out/var_{v}_{c}.err").read()[-500:])
PY
  done
done
