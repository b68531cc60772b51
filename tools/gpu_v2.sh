python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_heun.py -x -q > gpurun_out/pytest_heun.log 2>&1; echo "heun tests rc=$?"
S=$(date +%s); timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$? seconds=$(( $(date +%s) - S ))"
SEM_CHUNK=256 timeout 1200 python bench.py --no-orderings --no-orders --no-e2e --no-cpu > gpurun_out/bench_heun256.json 2> gpurun_out/bench_heun256.err; echo "bench256 rc=$?"
