#!/bin/bash
# Race / bounds checking of the asynchronous K7 / KH7 pipelines without compute-sanitizer
# (closed on this GPU pool).  Runs on a GPU box from the repo root:
#   /usr/local/graft/bin/gpurun --timeout 1800 -- 'bash tools/checked_build.sh'
# The checked library (-DSEM_CHECKED, built here or shipped in-tree) adds device asserts
# (stage meta == the chunk's descriptor, local indices / entry positions / slot ids in range,
# buffer capacities), poisons every shared-memory buffer before handing it back to its
# producer (stage, U^{n-1}/dt^2/M or (h/2)/M window, entry buffer), and inserts pseudo-random
# delays in producers and consumers.  A read that the mbarriers / named barriers did not order
# after its buffer's refill then sees NaN or an out-of-range index: an assert trap (SEM_E_CUDA)
# or a parity failure against the oracle.  Every run uses a capped persistent grid so each
# CTA walks many chunks (stage reuse, window hand-off, parity flips).
set -u
mkdir -p gpurun_out
LOG=gpurun_out/checked_build.log
: > $LOG
export SEM_LIB=paper_2104_08416_b200/libsem_checked.so
if [ ! -f $SEM_LIB ]; then
  python -c "from paper_2104_08416_b200 import build as b; b.build(force=True, out=b.PKG + '/libsem_checked.so', defines=['SEM_CHECKED'])" >> $LOG 2>&1 || exit 1
fi
echo "checked library: $SEM_LIB ($(strings $SEM_LIB | grep -c SEM_DCHECK) assert strings)" >> $LOG
for cap in 1 2 3; do
  echo "== pipeline cases, SEM_K7_GRID=$cap" >> $LOG
  SEM_K7_GRID=$cap SAN_STEPS=3 timeout 600 python tools/pipeline_cases.py >> $LOG 2>&1; echo "rc=$?" >> $LOG
done
echo "== GPU test-suite (parity, multirank, Heun, orders, strategies, ablation, chunks) with SEM_K7_GRID=4" >> $LOG
SEM_K7_GRID=4 timeout 1500 python -m pytest tests -m gpu -q -p no:randomly \
  --ignore=tests/test_gpu_multichunk.py >> $LOG 2>&1; echo "rc=$?" >> $LOG
echo "== many-chunks-per-CTA tests (their own caps 1-3)" >> $LOG
timeout 900 python -m pytest tests/test_gpu_multichunk.py -q >> $LOG 2>&1; echo "rc=$?" >> $LOG
echo "== the checker's own pin: a build whose consumers skip the stage waits on reused stages" >> $LOG
echo "   (SEM_INJECT_RACE) must be caught (expect a failure below)" >> $LOG
if [ -f paper_2104_08416_b200/libsem_checked_race.so ]; then
  SEM_LIB=paper_2104_08416_b200/libsem_checked_race.so SEM_K7_GRID=1 SAN_STEPS=3 timeout 300 \
    python tools/pipeline_cases.py lf >> $LOG 2>&1; echo "rc=$? (non-zero expected)" >> $LOG
fi
