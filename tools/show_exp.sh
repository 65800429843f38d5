#!/bin/bash
tag=$1
cat gpurun_out/${tag}_trace.txt; tail -3 gpurun_out/${tag}_pytest.txt
for w in c2 c3 c4; do python -c "
import json
try:
    d=json.load(open('gpurun_out/${tag}_bench_$w.json')); print('$w', round(d['us_per_layer_step'],2), d['stages_us'])
except Exception as e: print('$w failed', e)"; done
