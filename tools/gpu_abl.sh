set -x
python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_ablation.py -x -q > gpurun_out/pytest_abl.log 2>&1; echo "ablation tests rc=$?"
timeout 900 python bench.py --steps 1000 --no-e2e --no-cpu > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$?"
