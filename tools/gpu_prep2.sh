python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
SEM_TRACE=1 timeout 600 python tools/prep_trace_torch.py > gpurun_out/prep_trace3.log 2>&1; echo "rc=$?"
SEM_TRACE=1 timeout 600 python tools/prep_trace.py > gpurun_out/prep_trace4.log 2>&1; echo "rc=$?"
