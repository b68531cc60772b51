#!/bin/bash
# One GPU validation pass (run through gpurun from the repo root):
#   /usr/local/graft/bin/gpurun --timeout 2400 -- 'bash tools/gpu_validate.sh'
# build -> GPU tests -> smoke -> default bench (+ reference arm) -> ncu launch
# list and full K7 and K8 captures of the bench command (plain run first).
mkdir -p gpurun_out
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
S=$(date +%s); timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$? seconds=$(( $(date +%s) - S ))"
timeout 1200 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "reference rc=$?"
A="--steps 20 --warmup 3 --no-orderings --no-e2e --no-cpu --no-heun --no-orders --no-configs"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py $A > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k7_step -s 4 -c 1 -o gpurun_out/k7_full python bench.py --steps 6 --warmup 3 --no-orderings --no-e2e --no-cpu --no-heun --no-orders --no-configs > gpurun_out/ncu_full.log 2>&1; echo "ncu k7 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k8_fix -s 4 -c 1 -o gpurun_out/k8_full python bench.py --steps 6 --warmup 3 --no-orderings --no-e2e --no-cpu --no-heun --no-orders --no-configs > gpurun_out/ncu_k8.log 2>&1; echo "ncu k8 rc=$?"
