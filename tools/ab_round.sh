#!/bin/bash
# (SEM_K7_DYN exists only in the experiment build profiles/experiments/r2s4_k7_ticket_schedule.diff, removed from the library)
# Session-4 A/B on a GPU box: HEAD build (libsem_base.so) against the working tree's libsem.so
# on C4 and C3 (defaults), then the prefetched ticket schedule against round-robin.
mkdir -p gpurun_out
AB_TAG=_C4 timeout 900 bash tools/ab_lib.sh "libsem_base.so libsem.so" 2000
AB_TAG=_C3 timeout 600 bash tools/ab_lib.sh "libsem_base.so libsem.so" 2000 --config C3
timeout 900 bash tools/ab_env.sh SEM_K7_DYN "- 1" 2000
for f in gpurun_out/ab_lib_C4.txt gpurun_out/ab_lib_C3.txt gpurun_out/ab_SEM_K7_DYN.txt; do python tools/ab_summary.py $f; done
