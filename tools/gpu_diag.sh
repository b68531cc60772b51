python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python tools/e2e_diag.py > gpurun_out/e2e_diag.log 2>&1; echo "rc=$?"
