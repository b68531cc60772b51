python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "graph or c1_full or bitwise" > gpurun_out/pytest_graph.log 2>&1; echo "graph tests rc=$?"
for c in C1 C2 C4; do timeout 900 python bench.py --config $c --steps 2000 --no-orderings --no-e2e --no-cpu --no-heun --no-orders > gpurun_out/bench_graph_$c.json 2>gpurun_out/bench_graph_$c.err; echo "$c rc=$?"; done
for c in C1 C2; do SEM_GRAPH=0 timeout 900 python bench.py --config $c --steps 2000 --no-orderings --no-e2e --no-cpu --no-heun --no-orders > gpurun_out/bench_nograph_$c.json 2>gpurun_out/bench_nograph_$c.err; echo "$c nograph rc=$?"; done
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "all gpu tests rc=$?"
