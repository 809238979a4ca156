#!/bin/bash
# bench under named env settings: tools/ab_env.sh "NAME:VAR=v,VAR=v" ... (no CPU baseline)
for spec in "$@"; do
  name=${spec%%:*}; vars=${spec#*:}
  env $(echo "$vars" | tr ',' ' ') python bench.py --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/abn_$name.json 2> gpurun_out/abn_$name.err || tail -5 gpurun_out/abn_$name.err
  python -c "
import json; d=json.load(open('gpurun_out/abn_$name.json'))
print('%-12s %.4e samples/s  ms/step %.3f  draws %.3f' % ('$name', d['value'], d['ms_per_step'], d['kernel_ms_per_step']['draws']))"
done
