#!/bin/bash
# Bench every libvrs variant under paper_2505_10144_b200/variants (C2, no cpu baseline / e2e).
for lib in paper_2505_10144_b200/variants/libvrs_*.so; do
  n=$(basename $lib .so)
  VRS_LIB=$lib python bench.py --steps ${STEPS:-20} --warmup 3 --no-cpu-baseline --no-e2e ${EXTRA} > gpurun_out/var_$n.json 2>gpurun_out/var_$n.err
  python -c "
import json;d=json.loads(open('gpurun_out/var_$n.json').read().strip().splitlines()[-1])
print('$n', 'ms/frame', round(d['ms_per_step'],3), {k: round(v, 3) for k, v in d['stage_ms'].items()})" 2>/dev/null || tail -2 gpurun_out/var_$n.err
done
