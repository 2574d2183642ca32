#!/bin/bash
# Bench lines of every config (N=1) into gpurun_out/all_TAG_<config>.json.
# usage: tools/bench_all.sh TAG [configs...]
TAG=${1:-x}; shift
CFGS=${@:-c1 c2 c3 c4 c5 c6 c7}
mkdir -p gpurun_out
for c in $CFGS; do
  timeout 900 python bench.py --config $c ${EXTRA} > gpurun_out/all_${TAG}_$c.json 2> gpurun_out/all_${TAG}_$c.err
  echo "$c rc=$? $(tail -c 400 gpurun_out/all_${TAG}_$c.json | tr -d '\n' | cut -c1-200)"
done
