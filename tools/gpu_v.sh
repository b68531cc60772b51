python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "all gpu tests rc=$?"
SEM_TRACE=1 timeout 600 python tools/prep_trace_torch.py > gpurun_out/prep_trace5.log 2>&1; echo "trace rc=$?"
S=$(date +%s); timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$? seconds=$(( $(date +%s) - S ))"
