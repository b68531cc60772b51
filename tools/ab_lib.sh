#!/bin/bash
# A/B of two in-tree builds of the library on one bench workload, alternating runs (GPU box):
#   tools/ab_lib.sh "libsem_base.so libsem.so" [steps] [extra bench args...]
# Output: gpurun_out/ab_lib<tag>.txt (tools/ab_summary.py reads it); AB_TAG names the file.
libs=$1; steps=${2:-1000}; shift 2
out=gpurun_out/ab_lib${AB_TAG}.txt
mkdir -p gpurun_out
: > $out
for rep in 1 2; do
  for l in $libs; do
    SEM_LIB=$PWD/paper_2104_08416_b200/$l timeout 300 python bench.py --steps $steps --warmup 20 --no-orderings \
      --no-e2e --no-cpu --no-heun --no-orders --no-configs "$@" > gpurun_out/ab_run.json 2> gpurun_out/ab_run.err
    echo "lib=$l $*" >> $out
    grep "^{" gpurun_out/ab_run.json >> $out || tail -3 gpurun_out/ab_run.err >> $out
  done
done
