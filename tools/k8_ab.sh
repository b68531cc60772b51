#!/bin/bash
# K8 variants on a GPU box: parity tests with two shared nodes per thread (SEM_K8_NPT=2) and the
# descending node order (SEM_K8_REV=1), then alternating bench runs against the HEAD build
# (libsem_base.so) on C4 and C3.
mkdir -p gpurun_out
SEM_K8_NPT=2 SEM_K8_REV=1 timeout 900 python -m pytest tests -m gpu -x -q -k "parity or multichunk or knobs or graph or orders" \
  > gpurun_out/k8_pytest.log 2>&1; echo "npt2 tests rc=$?"
L=$PWD/paper_2104_08416_b200
for cfg in C4 C3; do
  out=gpurun_out/ab_k8_$cfg.txt; : > $out
  for rep in 1 2; do
    for v in "base - -" "new - -" "new 2 -" "new 2 1" "new - 1"; do
      set -- $v
      lib=$L/libsem.so; [ $1 = base ] && lib=$L/libsem_base.so
      env SEM_LIB=$lib $([ $2 != - ] && echo SEM_K8_NPT=$2) $([ $3 != - ] && echo SEM_K8_REV=$3) timeout 300 python bench.py --config $cfg \
        --steps 2000 --warmup 20 --no-orderings --no-e2e --no-cpu --no-heun --no-orders --no-configs > gpurun_out/ab_run.json 2> gpurun_out/ab_run.err
      echo "$1 NPT=$2 REV=$3" >> $out
      grep "^{" gpurun_out/ab_run.json >> $out || tail -3 gpurun_out/ab_run.err >> $out
    done
  done
  python tools/ab_summary.py $out
done
