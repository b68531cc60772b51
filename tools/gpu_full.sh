python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
free -g > gpurun_out/pytest_full.log
timeout 1200 python -m pytest tests/test_gpu_parity.py -k full_size -x -q --durations=5 >> gpurun_out/pytest_full.log 2>&1; echo "full tests rc=$?"
