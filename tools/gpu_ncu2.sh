python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
A="--steps 6 --warmup 3 --no-orderings --no-e2e --no-cpu"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_heun -s 6 -c 1 -o gpurun_out/heun_full python bench.py $A --no-orders > gpurun_out/ncu_heun.log 2>&1; echo "ncu heun rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k7_step -s 1 -c 1 -o gpurun_out/k7p5_full python bench.py --config C2 --steps 3 --warmup 3 --no-orderings --no-e2e --no-cpu --no-heun > gpurun_out/ncu_p5.log 2>&1; echo "ncu p5 rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches_full.csv python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu > gpurun_out/ncu_launch_full.log 2>&1; echo "ncu launches rc=$?"
