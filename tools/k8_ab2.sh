#!/bin/bash
# Session-4 K8 defaults (two nodes per thread, descending) on a GPU box: the whole GPU suite and
# smoke under the defaults, then K8 with 4 nodes per thread against the default.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu tests rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
SEM_K8_NPT=4 timeout 600 python -m pytest tests -m gpu -x -q -k "parity or multichunk or graph" > gpurun_out/k8_npt4_pytest.log 2>&1; echo "npt4 tests rc=$?"
for cfg in C4 C3; do
  timeout 900 bash tools/ab_env.sh SEM_K8_NPT "- 4 1" 2000 --config $cfg; cp gpurun_out/ab_SEM_K8_NPT.txt gpurun_out/ab_k8npt_$cfg.txt
  python tools/ab_summary.py gpurun_out/ab_k8npt_$cfg.txt
done
