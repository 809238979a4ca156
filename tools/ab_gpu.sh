#!/bin/bash
# A/B on the GPU box: short bench with an env toggle on and off (no CPU baseline)
#   usage: tools/ab_gpu.sh VAR [extra bench args]
VAR=$1; shift
for val in 0 1; do
  env $VAR=$val python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 "$@" > gpurun_out/ab_$val.json 2> gpurun_out/ab_$val.err || tail -20 gpurun_out/ab_$val.err
  python - "$VAR=$val" gpurun_out/ab_$val.json <<'PY'
import json, sys
d = json.load(open(sys.argv[2]))
print("%s value %.4e samples/s  ms/step %.3f  e2e %.3e  frac %.3f  kernels %s" % (
    sys.argv[1], d["value"], d["ms_per_step"], d["e2e"]["value"], d["roofline"]["frac"],
    {k: round(v, 3) for k, v in d["kernel_ms_per_step"].items()}))
PY
done
