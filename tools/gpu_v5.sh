python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"
for i in 1 2; do S=$(date +%s); timeout 1200 python bench.py > gpurun_out/bench_default_$i.json 2> gpurun_out/bench_default_$i.err; echo "bench rc=$? seconds=$(( $(date +%s) - S ))"; done
