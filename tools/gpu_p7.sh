python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
for g in 4 2 1; do
SEM_K7_G=$g timeout 900 python -m pytest tests/test_gpu_orders.py -x -q > gpurun_out/pytest_orders_g$g.log 2>&1; echo "G=$g orders tests rc=$?"
SEM_K7_G=$g timeout 900 python bench.py --steps 300 --no-orderings --no-e2e --no-cpu --no-heun > gpurun_out/bench_p7_g$g.json 2> gpurun_out/bench_p7_g$g.err; echo "G=$g bench rc=$?"
done
