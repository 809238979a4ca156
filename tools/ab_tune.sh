#!/bin/bash
# A/B on the GPU box: short config-2 bench under named tuning settings (no CPU baseline)
#   tools/ab_tune.sh "NAME:key=v,key=v" ...   e.g. "base:" "nosplit:eval_split=0"
for spec in "$@"; do
  name=${spec%%:*}; opts=${spec#*:}
  python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 --tune $(echo "$opts" | tr ',' ' ') \
      > gpurun_out/ab_$name.json 2> gpurun_out/ab_$name.err || tail -5 gpurun_out/ab_$name.err
  python -c "
import json; d=json.load(open('gpurun_out/ab_$name.json'))
print('%-12s %.4e samples/s  ms/step %.3f  e2e %.3e  frac %.3f  %s' % ('$name', d['value'], d['ms_per_step'],
      d['e2e']['value'], d['roofline']['frac'], {k: round(v, 3) for k, v in d['kernel_ms_per_step'].items()}))"
done
