python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k degenerate > gpurun_out/pytest_degen.log 2>&1; echo "degenerate rc=$?"
timeout 600 python bench.py --steps 20 --warmup 3 --no-orderings --no-e2e --no-cpu --no-heun --no-orders > gpurun_out/b_plain.json 2>&1; echo "plain rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 20 --warmup 3 --no-orderings --no-e2e --no-cpu --no-heun --no-orders > gpurun_out/ncu_launch_c4.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k7_step -s 4 -c 1 -o gpurun_out/k7_final python bench.py --steps 6 --warmup 3 --no-orderings --no-e2e --no-cpu --no-heun --no-orders > gpurun_out/ncu_k7_final.log 2>&1; echo "ncu k7 rc=$?"
