#!/bin/bash
# generic experiment round: GPU tests, clock64 traces of tc2 (c2, c3), stage times c2-c4
# usage: tools/gpu_exp.sh TAG [extra nvcc flags]
tag=$1; shift
mkdir -p gpurun_out
SALS_EXTRA_NVCC="-DSALS_TC_TRACE $*" python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
for w in c2 c3; do echo "== $tag $w"; timeout 300 python tools/trace_tc2.py $w; done > gpurun_out/${tag}_trace.txt 2>&1
SALS_EXTRA_NVCC="$*" python -m paper_2510_24273_b200.build --force > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/${tag}_pytest.txt
for w in c2 c3 c4; do timeout 300 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline --no-dense > gpurun_out/${tag}_bench_$w.json 2>gpurun_out/${tag}_bench_$w.err; done
