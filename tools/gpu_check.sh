set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 20 --warmup 3 --no-orderings --no-e2e --no-cpu > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k7_step -s 4 -c 1 -o gpurun_out/k7_full python bench.py --steps 6 --warmup 3 --no-orderings --no-e2e --no-cpu > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k8_fix -s 4 -c 1 -o gpurun_out/k8_full python bench.py --steps 6 --warmup 3 --no-orderings --no-e2e --no-cpu > gpurun_out/ncu_full8.log 2>&1; echo "ncu3 rc=$?"
