#!/bin/bash
# dev loop on the GPU box: parity subset + short bench (no CPU baseline)
python -m pytest tests/test_gpu_parity.py -q -x -k "sample_bit_exact or golden or tree_grams" 2>&1 | tail -3
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/bench_dev.json 2> gpurun_out/bench_dev.err || tail -20 gpurun_out/bench_dev.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/bench_dev.json"))
print("value %.3e samples/s  ms/step %.3f  e2e %.3e  draws frac %.3f  kernels %s  build %.3f ms (%.0f GB/s)" % (
    d["value"], d["ms_per_step"], d["e2e"]["value"], d["roofline"]["frac"], d["kernel_ms_per_step"],
    d["tree_build"]["ms_per_factor"], d["tree_build"]["achieved_gbs"]))
PY
python tools/prof_detail.py
