set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_orders.py -x -q > gpurun_out/pytest_orders.log 2>&1; echo "orders tests rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "all gpu tests rc=$?"
timeout 900 python bench.py --steps 300 --no-orderings --no-e2e --no-cpu --no-heun > gpurun_out/bench_orders.json 2> gpurun_out/bench_orders.err; echo "bench rc=$?"
