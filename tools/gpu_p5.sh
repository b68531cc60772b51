python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/dfma_peak tools/dfma_peak.cu && /tmp/dfma_peak > gpurun_out/dfma_peak.json; echo "dfma rc=$?"
timeout 900 python bench.py --steps 300 --no-orderings --no-e2e --no-cpu --no-heun > gpurun_out/bench_orders2.json 2> gpurun_out/bench_orders2.err; echo "bench rc=$?"
timeout 900 python -m pytest tests/test_gpu_orders.py -x -q > gpurun_out/pytest_orders.log 2>&1; echo "orders tests rc=$?"
