#!/bin/bash
# One-GPU evidence for the multi-GPU overlap: C4 on one rank with the
# chunk list split like the boundary / interior lists and a stand-in comm kernel (4 small CTAs
# holding their SMs for US microseconds, where NCCL's send/recv kernels would run) between
# them; SEM_COMM_SMS = SMs the interior K7 leaves free.  Run on a GPU box from the repo root.
US=${1:-20}
# SEM_OVERLAP_PROBE_SMEM_KB (environment): shared memory per stand-in CTA
out=gpurun_out/overlap_probe.txt
: >> $out
A="--steps 400 --warmup 10 --no-orderings --no-e2e --no-cpu --no-heun --no-orders --no-configs"
SEM_GRAPH=0 timeout 300 python bench.py $A > gpurun_out/op.json 2> gpurun_out/op.err
echo "no exchange (stream launches): $(python -c "import json;print(json.loads(open('gpurun_out/op.json').read().splitlines()[-1])['ms_per_step'])") ms/step" >> $out
echo "stand-in shared memory per CTA: ${SEM_OVERLAP_PROBE_SMEM_KB:-1} KB" >> $out
for r in ${SMS:-0 1 2 4 8}; do
  SEM_OVERLAP_PROBE_US=$US SEM_COMM_SMS=$r timeout 300 python bench.py $A > gpurun_out/op.json 2> gpurun_out/op.err
  echo "SEM_COMM_SMS=$r: $(python -c "import json;print(json.loads(open('gpurun_out/op.json').read().splitlines()[-1])['ms_per_step'])") ms/step (probe steps include a host sync each)" >> $out
  grep "overlap probe" gpurun_out/op.err | tail -1 >> $out
done
