#!/bin/bash
# A/B matrix on one bench workload, alternating runs (GPU box):
#   tools/ab_matrix.sh <out-tag> <steps> "lib1:ENV=v,ENV2=w lib2: ..." [extra bench args...]
# each entry: library file (in paper_2104_08416_b200/) then ':' and comma-separated env settings.
# Output: gpurun_out/ab_<tag>.txt (tools/ab_summary.py reads it).
tag=$1; steps=$2; entries=$3; shift 3
out=gpurun_out/ab_$tag.txt
mkdir -p gpurun_out
: > $out
for rep in 1 2; do
  for ent in $entries; do
    lib=${ent%%:*}; envs=${ent#*:}
    ( export SEM_LIB=$PWD/paper_2104_08416_b200/$lib
      for kv in ${envs//,/ }; do export "$kv"; done
      timeout 300 python bench.py --steps $steps --warmup 20 --no-orderings --no-e2e --no-cpu --no-heun --no-orders \
        --no-configs "$@" > gpurun_out/ab_run.json 2> gpurun_out/ab_run.err )
    echo "$ent $*" >> $out
    grep "^{" gpurun_out/ab_run.json >> $out || tail -3 gpurun_out/ab_run.err >> $out
  done
done
