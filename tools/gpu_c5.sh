python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
free -g > gpurun_out/c5.log; nvidia-smi --query-gpu=memory.total --format=csv >> gpurun_out/c5.log
S=$(date +%s); SEM_TEST_FULL_C5=1 timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k full_size_c5 --durations=3 >> gpurun_out/c5.log 2>&1; echo "c5 test rc=$? seconds=$(( $(date +%s) - S ))"
S=$(date +%s); timeout 1500 python bench.py --config C5 --steps 200 --no-orderings --no-e2e --no-cpu --no-heun --no-orders > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo "c5 bench rc=$? seconds=$(( $(date +%s) - S ))"
