#!/bin/bash
# One GPU iteration: parity tests, bench, launch list, one ncu --set full capture of a kernel.
# usage: tools/gpu_cycle.sh TAG [kernel_regex] [skip_tests]
TAG=${1:-x}; K=${2:-k_blend}; SKIP=${3:-0}
mkdir -p gpurun_out
if [ "$SKIP" != "1" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/tests_$TAG.log 2>&1
  tail -3 gpurun_out/tests_$TAG.log
fi
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
python -c "
import json;d=json.loads(open('gpurun_out/bench_$TAG.json').read().strip().splitlines()[-1])
print('ms/frame', round(d['ms_per_step'],3), 'fps', round(d['value'],1), {k:round(v,3) for k,v in d['stage_ms'].items()}, 'frac', round(d['roofline']['frac'],3))"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 3 --warmup 1 --no-cpu-baseline --no-e2e > /dev/null 2>&1
if [ -n "$K" ]; then
  ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_$TAG.log 2>&1
  tail -1 gpurun_out/ncu_$TAG.log
fi
