python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python bench.py --steps 20 --warmup 3 --no-orderings --no-e2e --no-cpu --no-heun --no-orders > gpurun_out/b_plain.json 2>&1; echo "plain rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k7_step -s 4 -c 1 -o gpurun_out/k7_waits python bench.py --steps 6 --warmup 3 --no-orderings --no-e2e --no-cpu --no-heun --no-orders > gpurun_out/ncu_k7_waits.log 2>&1; echo "ncu k7 rc=$?"
