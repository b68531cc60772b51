python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_heun.py -x -q > gpurun_out/pytest_heun5.log 2>&1; echo "heun tests rc=$?"
timeout 900 python bench.py --steps 300 --no-orderings --no-e2e --no-cpu --no-heun > gpurun_out/bench_heun5.json 2> gpurun_out/bench_heun5.err; echo "bench rc=$?"
