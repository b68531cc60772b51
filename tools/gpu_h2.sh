python __graft_entry__.py > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_gpu_heun.py -x -q > gpurun_out/pytest_heun.log 2>&1; echo "heun tests rc=$?"
for i in 1 2; do timeout 900 python bench.py --steps 500 --no-orderings --no-e2e --no-cpu --no-orders > gpurun_out/h2_$i.json 2>/dev/null; python -c "
import json; d=json.load(open('gpurun_out/h2_$i.json')); h=d['heun']; print('leap %.4f heun %.4f frac %.3f'%(d['ms_per_step'], h['ms_per_step'], h['roofline']['frac']))"; done
