python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_ablation.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_refac.log 2>&1; echo "tests rc=$?"
SEM_K7_G5=2 timeout 900 python -m pytest tests/test_gpu_orders.py -x -q > gpurun_out/pytest_p5g2.log 2>&1; echo "p5 g2 tests rc=$?"
SEM_K7_G5=2 timeout 900 python bench.py --steps 300 --no-orderings --no-e2e --no-cpu --no-heun > gpurun_out/bench_p5g2.json 2> gpurun_out/bench_p5g2.err; echo "bench rc=$?"
