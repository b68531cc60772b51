python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
A="--steps 1000 --no-orderings --no-e2e --no-cpu --no-heun --no-orders"
for m in fixed fit fixed fit; do SEM_K7_CSR=$m timeout 600 python bench.py $A > gpurun_out/csr_$m.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/csr_$m.json')); r=d['roofline']; print('$m', '%.4f'%d['ms_per_step'], 'k7 %.4f frac %.3f'%(r['avg_launch_ms'], r['frac']))"; done
SEM_K7_CSR=fit timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "c1_full or random_state or reduced or full_size" > gpurun_out/pytest_fit.log 2>&1; echo "fit tests rc=$?"
