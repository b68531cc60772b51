#!/bin/bash
# (SEM_K7_DYN exists only in the experiment build profiles/experiments/r2s4_k7_ticket_schedule.diff, removed from the library)
# Ticket-scheduled K7 (SEM_K7_DYN=1) on a GPU box: the K7 parity tests under it, then an
# alternating A/B against the round-robin default on C4 and C3.
mkdir -p gpurun_out
SEM_K7_DYN=1 timeout 900 python -m pytest tests -m gpu -x -q -k "parity or multichunk or multirank or knobs or graph" \
  > gpurun_out/dyn_pytest.log 2>&1; echo "dyn tests rc=$?"
timeout 900 bash tools/ab_env.sh SEM_K7_DYN "- 1" 2000; cp gpurun_out/ab_SEM_K7_DYN.txt gpurun_out/ab_dyn_C4.txt
timeout 600 bash tools/ab_env.sh SEM_K7_DYN "- 1" 2000 --config C3; cp gpurun_out/ab_SEM_K7_DYN.txt gpurun_out/ab_dyn_C3.txt
for f in gpurun_out/ab_dyn_C4.txt gpurun_out/ab_dyn_C3.txt; do python tools/ab_summary.py $f; done
