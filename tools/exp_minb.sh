#!/bin/bash
# projection launch-bounds variants (stage times + step from bench.py)
for mb in 2 1; do
  SALS_EXTRA_NVCC=-DSALS_PROJ_MINB=$mb python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
  for w in c2 c3 c4; do
    timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-dense 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w minb=$mb', round(d['us_per_layer_step'],1), d['stages_us'])"
  done
done > gpurun_out/exp_minb.log 2>&1
python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
