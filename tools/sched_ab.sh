#!/bin/bash
# (SEM_K7_DYN exists only in the experiment build profiles/experiments/r2s4_k7_ticket_schedule.diff, removed from the library)
# A/B of the K7 ticket schedule (SEM_K7_DYN) and K8's descending node order (SEM_K8_REV) on a
# GPU box: parity tests under both knobs, then alternating bench runs of the four combinations.
#   tools/sched_ab.sh [config] [steps]
cfg=${1:-C4}; steps=${2:-2000}
mkdir -p gpurun_out
if [ "$cfg" = "C4" ]; then
  SEM_K7_DYN=1 SEM_K8_REV=1 timeout 900 python -m pytest tests -m gpu -x -q -k "parity or multichunk or multirank or knobs or graph" \
    > gpurun_out/sched_pytest.log 2>&1; echo "dyn+rev tests rc=$?"
fi
out=gpurun_out/ab_sched_$cfg.txt
: > $out
for rep in 1 2 3; do
  for v in "0 0" "0 1" "1 0" "1 1"; do
    set -- $v
    SEM_K7_DYN=$1 SEM_K8_REV=$2 timeout 300 python bench.py --config $cfg --steps $steps --warmup 20 --no-orderings --no-e2e --no-cpu \
      --no-heun --no-orders --no-configs > gpurun_out/ab_run.json 2> gpurun_out/ab_run.err
    echo "DYN=$1 REV=$2" >> $out
    grep "^{" gpurun_out/ab_run.json >> $out || tail -3 gpurun_out/ab_run.err >> $out
  done
done
python tools/ab_summary.py $out
