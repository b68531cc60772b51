python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python bench.py --steps 300 --no-orderings --no-e2e --no-cpu --no-heun > gpurun_out/bench_orders46.json 2> gpurun_out/bench_orders46.err; echo "bench rc=$?"
