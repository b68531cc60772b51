set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"
timeout 600 python bench.py --steps 1000 --no-orderings --no-e2e --no-cpu --no-heun > gpurun_out/bench_fused.json 2> gpurun_out/bench_fused.err; echo "bench fused rc=$?"
SEM_NO_FUSE_K8=1 timeout 600 python bench.py --steps 1000 --no-orderings --no-e2e --no-cpu --no-heun > gpurun_out/bench_unfused.json 2> gpurun_out/bench_unfused.err; echo "bench unfused rc=$?"
timeout 600 python bench.py --config C3 --steps 1000 --no-orderings --no-e2e --no-cpu --no-heun > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3.err; echo "bench C3 rc=$?"
