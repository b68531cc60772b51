python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
nproc > gpurun_out/prep_trace.log; lscpu | grep -E "Model name|Socket|Core|Thread" >> gpurun_out/prep_trace.log
SEM_TRACE=1 timeout 600 python tools/prep_trace.py >> gpurun_out/prep_trace.log 2>&1; echo "rc=$?"
