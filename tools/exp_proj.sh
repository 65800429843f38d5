#!/bin/bash
# projection cluster-size sweep (stage times from bench.py)
for w in c2 c3; do for cs in 4 8 16; do
  SALS_PROJ_CS=$cs timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-dense 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w cs=$cs', round(d['us_per_layer_step'],1), d['stages_us'])"
done; done > gpurun_out/exp_proj.log 2>&1
