#!/bin/bash
# A/B of an environment knob on the default bench workload, alternating runs (on a GPU box):
#   tools/ab_env.sh VAR "v1 v2" [steps] [extra bench args...]
# a value "-" leaves VAR unset.  Output: gpurun_out/ab_VAR.txt (tools/ab_summary.py reads it).
var=$1; vals=$2; steps=${3:-1000}; shift 3
out=gpurun_out/ab_$var.txt
: > $out
for rep in 1 2; do
  for v in $vals; do
    if [ "$v" = "-" ]; then unset $var; else export $var=$v; fi
    timeout 300 python bench.py --steps $steps --warmup 20 --no-orderings --no-e2e --no-cpu --no-heun --no-orders --no-configs "$@" \
      > gpurun_out/ab_run.json 2> gpurun_out/ab_run.err
    echo "$var=$v" >> $out
    grep "^{" gpurun_out/ab_run.json >> $out || tail -3 gpurun_out/ab_run.err >> $out
  done
done
unset $var
