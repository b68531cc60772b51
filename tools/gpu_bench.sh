python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
S=$(date +%s); timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$? seconds=$(( $(date +%s) - S ))"
