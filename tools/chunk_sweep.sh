#!/bin/bash
# K7 chunk-size sweep on C4 (design experiment)
for B in ${BS:-128 192 256 512}; do
  SEM_CHUNK=$B python bench.py --steps 500 --warmup 10 --no-cpu --no-orderings --no-e2e > gpurun_out/sweep_B$B.json 2>gpurun_out/sweep_B$B.err || echo "B=$B failed"
done
