python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_chunks.py -x -q > gpurun_out/pytest_chunks.log 2>&1; echo "chunk tests rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "all gpu tests rc=$?"
SEM_TRACE=1 timeout 600 python tools/prep_trace.py > gpurun_out/prep_trace2.log 2>&1; echo "trace rc=$?"
timeout 900 python bench.py --no-orderings --no-heun --no-orders > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo "bench rc=$?"
