python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"
timeout 1200 python bench.py --no-orderings --no-e2e --no-cpu > gpurun_out/bench_h128.json 2> gpurun_out/bench_h128.err; echo "bench rc=$?"
SEM_CHUNK=256 timeout 1200 python bench.py --no-orderings --no-orders --no-e2e --no-cpu > gpurun_out/bench_h256.json 2> gpurun_out/bench_h256.err; echo "bench256 rc=$?"
