set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_heun.py -x -q > gpurun_out/pytest_heun.log 2>&1; echo "heun tests rc=$?"
timeout 600 python bench.py --steps 500 --no-orderings --no-e2e --no-cpu > gpurun_out/bench_heun.json 2> gpurun_out/bench_heun.err; echo "bench rc=$?"
SEM_CHUNK=128 timeout 600 python bench.py --steps 500 --no-orderings --no-e2e --no-cpu > gpurun_out/bench_heun128.json 2> gpurun_out/bench_heun128.err; echo "bench128 rc=$?"
