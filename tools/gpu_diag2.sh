python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
SEM_TRACE=1 timeout 900 python bench.py --no-cpu > gpurun_out/bench_trace.json 2> gpurun_out/bench_trace.err; echo "rc=$?"
