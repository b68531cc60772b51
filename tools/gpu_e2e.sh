python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python bench.py --no-orderings --no-heun --no-orders --no-cpu > gpurun_out/bench_e2e_only.json 2> gpurun_out/bench_e2e_only.err; echo "rc=$?"
timeout 900 python bench.py --no-cpu > gpurun_out/bench_e2e_full.json 2> gpurun_out/bench_e2e_full.err; echo "rc=$?"
