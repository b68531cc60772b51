python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests/test_gpu_orders.py -x -q > gpurun_out/pytest_orders46.log 2>&1; echo "orders tests rc=$?"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "all gpu tests rc=$?"
